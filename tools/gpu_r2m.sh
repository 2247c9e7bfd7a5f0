# round 2m: full GPU suite + sanitizers after the push combine / member cache; ncu of the long-row cluster kernels; default bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2m_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2m_pytest.log
timeout 2400 bash tools/gpu_sanitize.sh > gpurun_out/r2m_sanitize.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2m_rowcl_softmax python tools/long_rows_bench.py softmax_1024 --variant='{}' > gpurun_out/r2m_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2m_rowcl_ln python tools/long_rows_bench.py layernorm_1024 --variant='{}' >> gpurun_out/r2m_ncu.log 2>&1
timeout 600 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
