# round 2h: the online-softmax long-row pass — GPU tests, A/B against the two-pass forms, ncu
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "long or special or softmax or rows" > gpurun_out/r2h_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2h_pytest.log
timeout 900 python tools/long_rows_bench.py softmax layernorm > gpurun_out/r2h_longrows.jsonl 2> gpurun_out/r2h_longrows.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sfx_row(cl|mp)" -c 4 -o gpurun_out/r2h_longrows python tools/long_rows_bench.py softmax_1024 > gpurun_out/r2h_ncu.log 2>&1
