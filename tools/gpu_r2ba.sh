# LayerNorm long rows: variance folded in the mean's pass (cluster + multi-pass templates); parity, A/B, ncu
mkdir -p gpurun_out/r2ba
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bn or colbc or long or second_moment or row or layernorm or peer" > gpurun_out/r2ba/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ba/pytest.log
for i in 1 2; do
timeout 600 python tools/long_rows_bench.py layernorm > gpurun_out/r2ba/ln_one_pass.jsonl 2>&1
SFX_COLBC_TWO_PASS=1 timeout 600 python tools/long_rows_bench.py layernorm > gpurun_out/r2ba/ln_two_pass.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2ba/rowcl_ln python tools/long_rows_bench.py layernorm --variant='{}' > gpurun_out/r2ba/ncu.log 2>&1
tail -2 gpurun_out/r2ba/pytest.log; grep -E "FAIL|Error" gpurun_out/r2ba/pytest.log | head; cat gpurun_out/r2ba/ln_one_pass.jsonl gpurun_out/r2ba/ln_two_pass.jsonl
