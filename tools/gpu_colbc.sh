timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "long_and_odd" 2>&1 | tail -15
