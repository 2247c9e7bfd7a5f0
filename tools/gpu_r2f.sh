# round 2f: full GPU suite (ABI 3, self-checks, value map, pipelined host runs), autotune into the
# template parameter cache, C1 bench with / without the cache
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2f_pytest.log
timeout 1200 python tools/autotune.py gpurun_out/r2f_template_params.txt > gpurun_out/r2f_autotune.log 2>&1
for i in 1 2; do
  timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2f_C1_default_$i.json 2>/dev/null
  SFX_TEMPLATE_PARAMS=gpurun_out/r2f_template_params.txt timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2f_C1_tuned_$i.json 2>/dev/null
done
