mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fuse_dot or dot" > gpurun_out/r2an_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2an_pytest.log
timeout 900 python tools/layer_bench.py --config C5LF > gpurun_out/r2an_layer.json 2> gpurun_out/r2an_layer.err
timeout 1500 python tools/ab_kernels.py C5LF strategy=literal default > gpurun_out/r2an_ab.jsonl 2> gpurun_out/r2an_ab.err
