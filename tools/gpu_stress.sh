# widened random-graph stress through the reference-side binding (the reference's
# generator, inputs, compile_graph, interpret and values_close; fresh seeds)
for A in "random 31000 400 --fuse-dot-alternate" "random 32000 400" "random 33000 200 --fuse-dot-alternate --literal"; do
  timeout 2400 oracle/_ref/device_parity $A > gpurun_out/stress.log 2>&1; echo "$A rc=$?"; tail -1 gpurun_out/stress.log
done
