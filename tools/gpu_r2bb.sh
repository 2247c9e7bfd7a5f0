# full check after the second-moment folding: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out/r2bb
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bb/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bb/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bb/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bb/smoke.log
timeout 900 python bench.py > gpurun_out/r2bb/default.json 2> gpurun_out/r2bb/default.err
tail -3 gpurun_out/r2bb/pytest.log; grep -E "^FAILED|Error" gpurun_out/r2bb/pytest.log | head; tail -2 gpurun_out/r2bb/smoke.log; cut -c1-300 gpurun_out/r2bb/default.json
