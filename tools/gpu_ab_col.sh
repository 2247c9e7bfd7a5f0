# column template sweep on C3/C3b (stripes x residency x rows per iteration)
timeout 600 python tools/ab_kernels.py C3 default rows_per_cta=18,pipe_ctas_per_sm=1,items_per_thread=24 rows_per_cta=18,pipe_ctas_per_sm=1,items_per_thread=32 2>&1 | grep -v Warn | cut -c1-330
timeout 600 python tools/ab_kernels.py C3b default rows_per_cta=18,pipe_ctas_per_sm=1,items_per_thread=24 rows_per_cta=18,pipe_ctas_per_sm=1,items_per_thread=32 2>&1 | grep -v Warn | grep col_ | cut -c1-330
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "C3 or random or special or deterministic or nan or peer or odd" > gpurun_out/pytest_col.log 2>&1; tail -3 gpurun_out/pytest_col.log
