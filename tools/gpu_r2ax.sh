# colbc one-pass second moments: parity at the bench shapes (both forms, separate processes) + the new GPU tests
mkdir -p gpurun_out/r2ax
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bn or colbc or long_and_odd or peer or sync or second_moment" > gpurun_out/r2ax/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ax/pytest.log
timeout 900 python tools/colbc_check.py > gpurun_out/r2ax/check.jsonl 2> gpurun_out/r2ax/check.err; echo check rc=$?
tail -2 gpurun_out/r2ax/pytest.log; cat gpurun_out/r2ax/check.jsonl; tail -3 gpurun_out/r2ax/check.err
