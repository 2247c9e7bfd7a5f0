# two instances in flight for graphs > 512 MB: default bench (C5) twice, projection, 2-rank plumbing
mkdir -p gpurun_out
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r2as_default_$i.json 2> gpurun_out/r2as_default.err; done
timeout 1200 python tools/shard_projection.py > gpurun_out/r2as_proj.jsonl 2> gpurun_out/r2as_proj.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2as_c5_g2.json 2> gpurun_out/r2as_c5_g2.err
