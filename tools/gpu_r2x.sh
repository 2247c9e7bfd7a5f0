# round 2x: ncu of the widened templates after the round-2 changes (colbc ring + alternating passes, 16-CTA clusters)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2x_colbc_65536 python tools/long_rows_bench.py batchnorm_65536 --variant='{}' > gpurun_out/r2x_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2x_colbc_nhwc python tools/long_rows_bench.py batchnorm_nhwc --variant='{}' >> gpurun_out/r2x_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2x_rowcl_256 python tools/long_rows_bench.py softmax_256 --variant='{}' >> gpurun_out/r2x_ncu.log 2>&1
