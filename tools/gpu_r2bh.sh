# NCHW batch-norm: a thread-block cluster per channel (DSMEM combine) — parity, A/B vs one CTA per channel (pipe_stages=1), ncu
mkdir -p gpurun_out/r2bh
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "nchw or long_and_odd or channel_sums or colbc" > gpurun_out/r2bh/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bh/pytest.log
timeout 900 python tools/colbc_check.py > gpurun_out/r2bh/check.jsonl 2> gpurun_out/r2bh/check.err; echo check rc=$?
for i in 1 2; do
timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{}' >> gpurun_out/r2bh/nchw.jsonl 2>&1
timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{"pipe_stages": 1}' >> gpurun_out/r2bh/nchw_cta.jsonl 2>&1
done
timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{"items_per_thread": 12}' >> gpurun_out/r2bh/nchw_ur12.jsonl 2>&1
timeout 600 python tools/long_rows_bench.py batchnorm_nchw --variant='{"pipe_ctas_per_sm": 3}' >> gpurun_out/r2bh/nchw_cps3.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2bh/colbc_nchw python tools/long_rows_bench.py batchnorm_nchw_64 --variant='{}' > gpurun_out/r2bh/ncu.log 2>&1
tail -2 gpurun_out/r2bh/pytest.log; grep -E "^FAILED" gpurun_out/r2bh/pytest.log | head; grep nchw gpurun_out/r2bh/check.jsonl | cut -c1-160; tail -3 gpurun_out/r2bh/check.err; cat gpurun_out/r2bh/nchw*.jsonl
