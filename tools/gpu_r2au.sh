# final check with the pruned kernel cache (kernels not prebuilt compile on the box)
mkdir -p gpurun_out/r2au
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2au/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2au/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2au/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2au/smoke.log
timeout 900 python bench.py > gpurun_out/r2au/default.json 2> gpurun_out/r2au/default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2au/reference.json 2> gpurun_out/r2au/reference.err
