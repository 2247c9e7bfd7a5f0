timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "long_and_odd or tma or configs_small" > gpurun_out/pytest_gpu3.log 2>&1; tail -3 gpurun_out/pytest_gpu3.log
timeout 600 python tools/ab_kernels.py C5 default rows_per_cta=4 rows_per_cta=2 threads_per_row=16 threads_per_row=64 2>&1 | grep -E '"h1"|"probs_d"'
timeout 300 python tools/ab_kernels.py C1 default rows_per_cta=4 threads_per_row=64 threads_per_row=128 2>&1 | tail -4
timeout 300 python tools/ab_kernels.py C2 default rows_per_cta=4 threads_per_row=16 threads_per_row=64 2>&1 | tail -4
