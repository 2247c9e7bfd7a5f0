for C in C1 C2 C5; do timeout 300 python tools/ab_kernels.py $C row_pipeline=1 row_pipeline=2 2>&1 | tail -12; done
AB_SIZE=small timeout 300 python tools/ab_kernels.py C1 row_pipeline=1 row_pipeline=2 2>&1 | tail -4
AB_SIZE=small timeout 300 python tools/ab_kernels.py C5 row_pipeline=2 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu6.log 2>&1; tail -3 gpurun_out/pytest_gpu6.log
for C in C5 C1; do timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench6_$C.json 2> gpurun_out/bench6_$C.err; python -c "import json,sys; d=json.load(open('gpurun_out/bench6_$C.json')); print('$C', round(d['value']), round(d['pct_of_peak'],1), d['clocks']['sm_mhz'], d['clocks']['reasons']); [print('   ', k['group'], k['strategy'], round(k['gbs']), k['regs'], round(k['ms']*1000,1)) for k in d['per_kernel']]" || tail -5 gpurun_out/bench6_$C.err; done
