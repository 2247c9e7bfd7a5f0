# split colbc: clusters per channel from 37 channels (K=64: [32,64,112,112]) vs stripes + grid barrier (pipe_stages=1)
mkdir -p gpurun_out/r2bi
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "nchw or channel_sums" > gpurun_out/r2bi/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bi/pytest.log
for i in 1 2; do
timeout 600 python tools/long_rows_bench.py batchnorm_nchw_32 --variant='{}' >> gpurun_out/r2bi/nchw.jsonl 2>&1
timeout 600 python tools/long_rows_bench.py batchnorm_nchw_32 --variant='{"pipe_stages": 1}' >> gpurun_out/r2bi/nchw_stripes.jsonl 2>&1
done
timeout 900 python tools/colbc_check.py > gpurun_out/r2bi/check.jsonl 2> gpurun_out/r2bi/check.err; echo check rc=$?
tail -2 gpurun_out/r2bi/pytest.log; grep -E "^FAILED" gpurun_out/r2bi/pytest.log | head; grep nchw_32 gpurun_out/r2bi/check.jsonl | cut -c1-150; cat gpurun_out/r2bi/nchw*.jsonl
