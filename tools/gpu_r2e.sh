# round 2e: C1 row-template A/B with back-to-back timing; ncu of the 1-CTA/SM TMA-staged variant and the tiled transpose
mkdir -p gpurun_out
timeout 900 python tools/ab_kernels.py C1 default threads_per_row=64 threads_per_row=128 pipe_ctas_per_sm=5 pipe_ctas_per_sm=6 threads_per_row=64,pipe_ctas_per_sm=8 rows_per_cta=4 row_pipeline=2,pipe_warps=28,pipe_stages=2,pipe_ctas_per_sm=1 row_pipeline=2,pipe_warps=14,pipe_stages=2,pipe_ctas_per_sm=2 row_pipeline=2,pipe_warps=7,pipe_stages=2,pipe_ctas_per_sm=4 > gpurun_out/r2e_ab_C1.jsonl 2> gpurun_out/r2e_ab_C1.err
timeout 600 python tools/ab_kernels.py C4t default items_per_thread=2 > gpurun_out/r2e_ab_C4t.jsonl 2> gpurun_out/r2e_ab_C4t.err
timeout 600 python tools/ab_kernels.py C4 default items_per_thread=2 items_per_thread=4 > gpurun_out/r2e_ab_C4.jsonl 2> gpurun_out/r2e_ab_C4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowp" -s 3 -c 1 -o gpurun_out/r2e_C1_rowp python tools/ab_kernels.py C1 row_pipeline=2,pipe_warps=28,pipe_stages=2,pipe_ctas_per_sm=1 > gpurun_out/r2e_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_mapt" -s 3 -c 1 -o gpurun_out/r2e_C4t python tools/ab_kernels.py C4t default > gpurun_out/r2e_ncu2.log 2>&1
