# C3b column kernel with writes: residency x rows in flight
mkdir -p gpurun_out
timeout 900 python tools/ab_kernels.py C3b default pipe_ctas_per_sm=3,items_per_thread=12 pipe_ctas_per_sm=4,items_per_thread=8 pipe_ctas_per_sm=4,items_per_thread=12 pipe_ctas_per_sm=1,items_per_thread=32 > gpurun_out/r2aa_C3b.jsonl 2> gpurun_out/r2aa.err
