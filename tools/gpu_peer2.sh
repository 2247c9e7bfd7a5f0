python tools/peer_overhead.py C3 2>&1 | grep -v Warn
python tools/peer_overhead.py C3b 2>&1 | grep -v Warn
bash tools/gpu_multirank.sh 2>&1 | tail -6
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --config C3 --no-cpu-baseline > gpurun_out/mr_c3_peer.json 2> gpurun_out/mr_c3_peer.err; echo rc=$?; tail -c 300 gpurun_out/mr_c3_peer.json
