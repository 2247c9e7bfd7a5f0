# round 2l: cluster combine by st.async push + per-level mbarriers (no per-level cluster barriers), parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long_and_odd or special_rows" > gpurun_out/r2l_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2l_pytest.log
timeout 600 python tools/long_rows_bench.py softmax layernorm > gpurun_out/r2l_longrows.jsonl 2> gpurun_out/r2l_longrows.err
SFX_CLUSTER_BARRIER_COMBINE=1 timeout 600 python tools/long_rows_bench.py softmax layernorm > gpurun_out/r2l_longrows_bar.jsonl 2>> gpurun_out/r2l_longrows.err
