# round 2s: C1 row-template granularity sweep (rows per CTA 1/2/4, threads per row 64)
mkdir -p gpurun_out
timeout 900 python tools/ab_kernels.py C1 default rows_per_cta=1 rows_per_cta=2 rows_per_cta=4 threads_per_row=64,rows_per_cta=1 threads_per_row=64,rows_per_cta=2 threads_per_row=128,rows_per_cta=1 default > gpurun_out/r2s_ab_C1.jsonl 2> gpurun_out/r2s_ab_C1.err
