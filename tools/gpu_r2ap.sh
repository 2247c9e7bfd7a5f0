mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fuse_dot or dot or encoder or reference_suites or fixture" > gpurun_out/r2ap_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ap_pytest.log
timeout 900 python tools/layer_bench.py --config C5LF > gpurun_out/r2ap_layer.json 2> gpurun_out/r2ap_layer.err
timeout 900 python tools/dot_check.py > gpurun_out/r2ap_dot.jsonl 2> gpurun_out/r2ap_dot.err
timeout 900 oracle/_ref/device_parity random 45000 300 --fuse-dot-alternate > gpurun_out/r2ap_stress.log 2>&1; echo rc=$? >> gpurun_out/r2ap_stress.log
