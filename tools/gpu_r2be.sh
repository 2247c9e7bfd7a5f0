# NCHW batch-norm: the parity test at the +2 offset; the literal tier's time at the bench shape (one block, the reference's plan)
mkdir -p gpurun_out/r2be
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "nchw or long_and_odd or channel_sums or colbc" > gpurun_out/r2be/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2be/pytest.log
timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{"strategy": "literal"}' > gpurun_out/r2be/nchw_literal.jsonl 2>&1
tail -2 gpurun_out/r2be/pytest.log; grep -E "^FAILED" gpurun_out/r2be/pytest.log | head; cat gpurun_out/r2be/nchw_literal.jsonl | tail -3
