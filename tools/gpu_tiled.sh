timeout 300 python tools/ab_kernels.py C4t default items_per_thread=1 default items_per_thread=1 2>&1 | grep -v Warn | cut -c1-260
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "C4t or head_split or encoder" 2>&1 | tail -2
