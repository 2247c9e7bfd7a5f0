# packed fp32x2 SIMT matmul: bit-exactness tests, dot_check, layer bench, encoder-layer + reference suites
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "dot or encoder or reference_suites or fixture" > gpurun_out/r2ae_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ae_pytest.log
timeout 900 python tools/dot_check.py > gpurun_out/r2ae_dot.jsonl 2> gpurun_out/r2ae_dot.err
SFX_DOT_PACKED=0 timeout 900 python tools/dot_check.py > gpurun_out/r2ae_dot_old.jsonl 2>> gpurun_out/r2ae_dot.err
timeout 900 python tools/layer_bench.py > gpurun_out/r2ae_layer.json 2> gpurun_out/r2ae_layer.err
