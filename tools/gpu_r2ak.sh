# fuse_dot groups as prologue-fused dot kernels: parity (C5LF small, bit-exact vs literal, reference suites), layer bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fuse_dot or encoder or reference_suites or fixture or dot" > gpurun_out/r2ak_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ak_pytest.log
timeout 900 python tools/layer_bench.py --config C5LF > gpurun_out/r2ak_layer.json 2> gpurun_out/r2ak_layer.err
timeout 900 oracle/_ref/device_parity random 44000 300 --fuse-dot-alternate > gpurun_out/r2ak_stress.log 2>&1; echo rc=$? >> gpurun_out/r2ak_stress.log
