# round 2n: colbc passes alternate direction (L2 reuse across passes), parity + A/B + ncu of colbc
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "bn or colbc or batchnorm or peer" > gpurun_out/r2n_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2n_pytest.log
timeout 600 python tools/long_rows_bench.py batchnorm > gpurun_out/r2n_bn.jsonl 2> gpurun_out/r2n_bn.err
SFX_COLBC_FORWARD=1 timeout 600 python tools/long_rows_bench.py batchnorm > gpurun_out/r2n_bn_fwd.jsonl 2>> gpurun_out/r2n_bn.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2n_colbc_65536 python tools/long_rows_bench.py batchnorm_65536 --variant='{}' > gpurun_out/r2n_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2n_colbc_nhwc python tools/long_rows_bench.py batchnorm_nhwc --variant='{}' >> gpurun_out/r2n_ncu.log 2>&1
