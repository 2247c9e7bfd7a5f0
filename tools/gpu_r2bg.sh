# final check after the second-moment folding and the NCHW template: GPU suite, smoke, default + reference arm, every config's bench line
mkdir -p gpurun_out/r2bg
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bg/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bg/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bg/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bg/smoke.log
timeout 900 python bench.py > gpurun_out/r2bg/default.json 2> gpurun_out/r2bg/default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2bg/reference.json 2> gpurun_out/r2bg/reference.err
bash tools/gpu_benches.sh > gpurun_out/r2bg/benches.log 2>&1
tail -3 gpurun_out/r2bg/pytest.log; cat gpurun_out/r2bg/smoke.log | tail -2; cat gpurun_out/r2bg/default.json | cut -c1-400
