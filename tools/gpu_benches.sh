# every config's bench line (device path + e2e), then the default line with the CPU baseline
mkdir -p gpurun_out/bench
for C in C5 C1 C2 C3 C3b C4 C4b C4t; do
  timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench/$C.json 2> gpurun_out/bench/$C.err
  python -c "import json; d=json.load(open('gpurun_out/bench/$C.json')); print('$C', round(d['value']), round(d['pct_of_peak'],1), 'e2e', round(d['e2e']['value'],1), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons']); [print('   ', k['group'], k['strategy'], round(k['gbs']), k['regs'], round(k['ms']*1000,1)) for k in d['per_kernel']]" || tail -3 gpurun_out/bench/$C.err
done
timeout 600 python bench.py > gpurun_out/bench/default.json 2> gpurun_out/bench/default.err; tail -c 700 gpurun_out/bench/default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench/reference.json 2> gpurun_out/bench/reference.err; tail -c 500 gpurun_out/bench/reference.json
