# packed fp32x2 SIMT matmul incl. 128x64 tiles: tests, dot_check, layer bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "dot or encoder or reference_suites or fixture" > gpurun_out/r2ag_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ag_pytest.log
timeout 900 python tools/dot_check.py > gpurun_out/r2ag_dot.jsonl 2> gpurun_out/r2ag_dot.err
timeout 900 python tools/layer_bench.py > gpurun_out/r2ag_layer.json 2> gpurun_out/r2ag_layer.err
