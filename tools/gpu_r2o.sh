# round 2o: colbc stripe passes through a per-thread cp.async ring — parity (incl. SyncBatchNorm peers) + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "bn or colbc or batchnorm or peer or long_and_odd" > gpurun_out/r2o_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2o_pytest.log
timeout 900 python tools/long_rows_bench.py batchnorm > gpurun_out/r2o_bn.jsonl 2> gpurun_out/r2o_bn.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2o_colbc_65536 python tools/long_rows_bench.py batchnorm_65536 --variant='{}' > gpurun_out/r2o_ncu.log 2>&1
