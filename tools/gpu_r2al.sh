mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fuse_dot or encoder or reference_suites or fixture or dot" > gpurun_out/r2al_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2al_pytest.log
timeout 900 python tools/layer_bench.py --config C5LF > gpurun_out/r2al_layer.json 2> gpurun_out/r2al_layer.err
