# round 2q: C3b bench line (missing from the round-2 table), resident-row tests, launch log test
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "tma_row_pipeline or resident or launch_log" > gpurun_out/r2q_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2q_pytest.log
for i in 1 2; do timeout 600 python bench.py --config C3b --no-cpu-baseline > gpurun_out/r2q_C3b_$i.json 2> gpurun_out/r2q_C3b_$i.err; done
timeout 600 python tools/ab_kernels.py C3b default > gpurun_out/r2q_ab_C3b.jsonl 2> gpurun_out/r2q_ab_C3b.err
timeout 600 python tools/ab_kernels.py C3 default > gpurun_out/r2q_ab_C3.jsonl 2>> gpurun_out/r2q_ab_C3b.err
