# round 2w: long-row cluster template — vectors in flight per thread (items_per_thread) and threads per CTA
mkdir -p gpurun_out
for v in '{"items_per_thread": 2}' '{"items_per_thread": 8}' '{"items_per_thread": 16}' '{"threads_per_row": 256}' '{"threads_per_row": 1024}' '{}'; do
  timeout 300 python tools/long_rows_bench.py layernorm_1024 softmax_1024 --variant="$v" >> gpurun_out/r2w_longrows.jsonl 2>> gpurun_out/r2w.err
done
