# Cross-rank peer-memory column combine on the 1-GPU box: GPU tests (2 processes
# sharing cuda:0 through CUDA IPC) + a 2-rank C3 bench smoke (gloo plumbing).
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -x > gpurun_out/peer_pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/peer_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --config C3 --no-cpu-baseline > gpurun_out/mr_c3_peer.json 2> gpurun_out/mr_c3_peer.err; echo rc=$?; tail -c 600 gpurun_out/mr_c3_peer.json; tail -5 gpurun_out/mr_c3_peer.err
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 50 > gpurun_out/c3_1.json 2>gpurun_out/c3_1.err; python -c "import json; d=json.load(open('gpurun_out/c3_1.json')); print('C3 N=1', round(d['value']), [ (k['group'], round(k['gbs'])) for k in d['per_kernel']])"
