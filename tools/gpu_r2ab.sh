# multi-rank plumbing after the late round-2 changes (gloo ranks time-slicing one GPU; not a timing)
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_c1_g2.json 2> gpurun_out/r2ab_c1_g2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_c3_g2.json 2> gpurun_out/r2ab_c3_g2.err
timeout 900 python bench.py --gpus 4 --dist-backend gloo --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_c5_g4.json 2> gpurun_out/r2ab_c5_g4.err
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q > gpurun_out/r2ab_peer.log 2>&1; echo rc=$? >> gpurun_out/r2ab_peer.log
