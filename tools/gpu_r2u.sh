# round 2u: C1 with the tuned row granularity (template parameter cache): parity + bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "C1 or host_stream or template or smoke or resident" > gpurun_out/r2u_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2u_pytest.log
for i in 1 2; do timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r2u_C1_$i.json 2> gpurun_out/r2u_C1.err; done
