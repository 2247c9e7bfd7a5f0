# round 2k: long-row cluster template caching exp(x - max) over the input slice (row_pipeline=5 = recompute), parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long_and_odd or special_rows" > gpurun_out/r2k_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2k_pytest.log
timeout 600 python tools/long_rows_bench.py softmax layernorm > gpurun_out/r2k_longrows.jsonl 2> gpurun_out/r2k_longrows.err
