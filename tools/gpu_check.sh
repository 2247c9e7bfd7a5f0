# GPU box round check: parity suite, bench for every config, then profiles.
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for C in C5 C1 C2 C3 C3b C4 C4b; do
  timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_$C.json')); print('$C', round(d['value']), round(d['pct_of_peak'],1), 'inflight', d['config']['instances_in_flight'], d['clocks']['sm_mhz'], d['clocks']['reasons']); [print('   ', k['group'], k['strategy'], round(k['gbs']), k['regs'], round(k['ms']*1000,1)) for k in d['per_kernel']]" || tail -5 gpurun_out/bench_$C.err
done
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
