timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/ab_kernels.py C4t default items_per_thread=4 2>&1 | tail -2
for C in C5 C4t; do
  timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_$C.json')); print('$C', round(d['value']), round(d['pct_of_peak'],1), 'inflight', d['config']['instances_in_flight'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1)); [print('   ', k['group'], k['strategy'], round(k['gbs']), k['regs'], round(k['ms']*1000,1)) for k in d['per_kernel']]" || tail -5 gpurun_out/bench_$C.err
done
