# split colbc (clusters per channel): rows-in-flight and residency sweep
mkdir -p gpurun_out/r2bl
for V in '{}' '{"items_per_thread": 4}' '{"items_per_thread": 12}' '{"items_per_thread": 16}' '{"pipe_ctas_per_sm": 3}' '{"pipe_ctas_per_sm": 4}' '{}'; do
  timeout 300 python tools/long_rows_bench.py batchnorm_nchw --variant="$V" >> gpurun_out/r2bl/sweep.jsonl 2>&1
done
cat gpurun_out/r2bl/sweep.jsonl
