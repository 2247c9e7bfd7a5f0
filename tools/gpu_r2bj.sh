# final check after the second-moment folding and the NCHW template: GPU suite, smoke, default + reference arm, every config's bench line
mkdir -p gpurun_out/r2bj
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bj/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bj/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bj/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bj/smoke.log
timeout 900 python bench.py > gpurun_out/r2bj/default.json 2> gpurun_out/r2bj/default.err
timeout 900 python bench.py --impl reference > gpurun_out/r2bj/reference.json 2> gpurun_out/r2bj/reference.err
bash tools/gpu_benches.sh > gpurun_out/r2bj/benches.log 2>&1
tail -3 gpurun_out/r2bj/pytest.log; cat gpurun_out/r2bj/smoke.log | tail -2; cat gpurun_out/r2bj/default.json | cut -c1-400
