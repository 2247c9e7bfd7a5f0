# round 2d: new tests (value map, per-stream intermediates, pipelined host runs, perflib fixpoint),
# default bench with the pipelined e2e, C1 row-template A/B + ncu of the register and TMA row kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "full_value_map or intermediates or pipelined or perflib or concurrent" > gpurun_out/r2d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
timeout 600 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_C1.json 2> gpurun_out/r2d_bench_C1.err
timeout 900 python tools/ab_kernels.py C1 default threads_per_row=64 threads_per_row=128 threads_per_row=256 rows_per_cta=4 row_pipeline=2 row_pipeline=2,pipe_warps=16,pipe_stages=3,pipe_ctas_per_sm=1 row_pipeline=2,pipe_warps=8,pipe_stages=2 > gpurun_out/r2d_ab_C1.jsonl 2> gpurun_out/r2d_ab_C1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_row" -c 3 -o gpurun_out/r2d_C1 python tools/ab_kernels.py C1 default row_pipeline=2 threads_per_row=128 > gpurun_out/r2d_ncu.log 2>&1
