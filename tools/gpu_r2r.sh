mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_launch_log.py -m gpu -q > gpurun_out/r2r_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2r_pytest.log
