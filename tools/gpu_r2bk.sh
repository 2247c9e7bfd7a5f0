# fresh random-graph stress after the last lowering changes (colbc second moments, split colbc): the reference's
# generator / compile_graph / interpret / values_close through the reference-side binding
mkdir -p gpurun_out/r2bk
for A in "random 51000 400 --fuse-dot-alternate" "random 52000 400"; do
  timeout 1500 oracle/_ref/device_parity $A > gpurun_out/r2bk/stress_$(echo $A | cut -d' ' -f2).log 2>&1; echo "$A rc=$?"; tail -1 gpurun_out/r2bk/stress_$(echo $A | cut -d' ' -f2).log
done
