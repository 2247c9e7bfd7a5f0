# batch-norm over NCHW: the split colbc template — parity (tests, bench shapes vs the fp64 oracle), timing, ncu
mkdir -p gpurun_out/r2bd
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bn or colbc or long_and_odd or second_moment or nchw" > gpurun_out/r2bd/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bd/pytest.log
timeout 900 python tools/colbc_check.py > gpurun_out/r2bd/check.jsonl 2> gpurun_out/r2bd/check.err; echo check rc=$?
timeout 600 python tools/long_rows_bench.py batchnorm_nchw > gpurun_out/r2bd/nchw.jsonl 2>&1
SFX_COLBC_TWO_PASS=1 timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{}' > gpurun_out/r2bd/nchw_two_pass.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2bd/colbc_nchw python tools/long_rows_bench.py batchnorm_nchw_64 --variant='{}' > gpurun_out/r2bd/ncu.log 2>&1
tail -2 gpurun_out/r2bd/pytest.log; grep -E "^FAILED|Error|assert" gpurun_out/r2bd/pytest.log | head -8; cut -c1-200 gpurun_out/r2bd/check.jsonl; tail -3 gpurun_out/r2bd/check.err; cat gpurun_out/r2bd/nchw.jsonl gpurun_out/r2bd/nchw_two_pass.jsonl
