# colbc second moments: non-finite columns through both forms; parity at the bench shapes; timing unchanged
mkdir -p gpurun_out/r2az
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bn or colbc or long_and_odd or peer or sync or second_moment" > gpurun_out/r2az/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2az/pytest.log
timeout 900 python tools/colbc_check.py > gpurun_out/r2az/check.jsonl 2> gpurun_out/r2az/check.err; echo check rc=$?
timeout 600 python tools/long_rows_bench.py batchnorm --variant='{}' > gpurun_out/r2az/one_pass.jsonl 2>&1
tail -2 gpurun_out/r2az/pytest.log; grep -E "FAIL|Error" gpurun_out/r2az/pytest.log | head; cut -c1-150 gpurun_out/r2az/check.jsonl; cat gpurun_out/r2az/one_pass.jsonl
