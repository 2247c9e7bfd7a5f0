# round-end check: GPU suite, smoke, every config's bench line, default + reference arm, 2-rank smoke
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/gpu_benches.sh 2>&1 | grep -v "^ " | tail -12
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/mr_c5.json 2> gpurun_out/mr_c5.err; echo "2-rank C5 rc=$?"; tail -c 300 gpurun_out/mr_c5.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --config C3 --no-cpu-baseline > gpurun_out/mr_c3.json 2> gpurun_out/mr_c3.err; echo "2-rank C3 (peer combine) rc=$?"; tail -c 300 gpurun_out/mr_c3.json
