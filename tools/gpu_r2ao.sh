# final round-2 check after the packed / prologue matmuls: full GPU suite, smoke, default bench + reference, sanitizers (incl. C5L / C5LF)
mkdir -p gpurun_out/r2ao
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2ao/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ao/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ao/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2ao/smoke.log
timeout 900 python bench.py > gpurun_out/r2ao/default.json 2> gpurun_out/r2ao/default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2ao/reference.json 2> gpurun_out/r2ao/reference.err
timeout 3000 bash tools/gpu_sanitize.sh > gpurun_out/r2ao/sanitize.log 2>&1
