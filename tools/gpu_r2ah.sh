# random-graph stress through the reference-side binding after the packed matmul (fresh seeds)
mkdir -p gpurun_out
for A in "random 41000 400 --fuse-dot-alternate" "random 42000 400" "random 43000 200 --fuse-dot-alternate --literal"; do
  timeout 2400 oracle/_ref/device_parity $A > gpurun_out/r2ah_stress.log 2>&1; echo "$A rc=$?" >> gpurun_out/r2ah_stress.txt; tail -2 gpurun_out/r2ah_stress.log >> gpurun_out/r2ah_stress.txt
done
