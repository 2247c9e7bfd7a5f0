mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fuse_dot or encoder or reference_suites or fixture or dot" > gpurun_out/r2am_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2am_pytest.log
timeout 900 python tools/layer_bench.py --config C5LF > gpurun_out/r2am_layer.json 2> gpurun_out/r2am_layer.err
timeout 900 python tools/dot_check.py > gpurun_out/r2am_dot.jsonl 2> gpurun_out/r2am_dot.err
