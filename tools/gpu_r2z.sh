# round 2z: final round-2 check — full GPU suite, smoke, every bench line, reference arm, ncu profiles, sanitizers
mkdir -p gpurun_out/r2z
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2z/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2z/smoke.log
timeout 900 python bench.py > gpurun_out/r2z/default.json 2> gpurun_out/r2z/default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2z/reference.json 2> gpurun_out/r2z/reference.err
for C in C1 C2 C3 C3b C4 C4b C4t; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2z/$C.json 2> gpurun_out/r2z/$C.err
done
timeout 1800 bash profiles/run_profiles.sh r02f > gpurun_out/r2z/profiles.log 2>&1
timeout 2400 bash tools/gpu_sanitize.sh > gpurun_out/r2z/sanitize.log 2>&1
