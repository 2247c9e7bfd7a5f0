# round 2g: multi-rank plumbing on one GPU (gloo, strong sharding), round-2 ncu captures, sanitizers incl. the new host path
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c5_g2.json 2> gpurun_out/r2g_c5_g2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c3_g2.json 2> gpurun_out/r2g_c3_g2.err
timeout 600 python bench.py --gpus 4 --dist-backend gloo --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c1_g4.json 2> gpurun_out/r2g_c1_g4.err
timeout 1800 bash profiles/run_profiles.sh r02 > gpurun_out/r2g_profiles.log 2>&1
timeout 2400 bash tools/gpu_sanitize.sh > gpurun_out/r2g_sanitize.log 2>&1
