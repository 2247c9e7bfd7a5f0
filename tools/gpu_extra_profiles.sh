ncu --set full --clock-control none -k regex:sfx_rowcl_ -s 2 -c 1 -o gpurun_out/x_rowcl python tools/long_rows_bench.py softmax_1024 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:sfx_rowmp_ -s 2 -c 1 -o gpurun_out/x_rowmp python tools/long_rows_bench.py softmax_256 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:sfx_colbc_ -s 2 -c 1 -o gpurun_out/x_colbc python tools/long_rows_bench.py batchnorm_65536 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:sfx_colbc_ -s 2 -c 1 -o gpurun_out/x_colbc_nhwc python tools/long_rows_bench.py batchnorm_nhwc > /dev/null 2>&1
ls gpurun_out/x_*.ncu-rep
