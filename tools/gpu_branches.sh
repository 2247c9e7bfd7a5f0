# A/B: independent groups on concurrent CUDA-graph branches (device path)
for B in 1 0 1 0; do
  SFX_GRAPH_BRANCHES=$B timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 100 > gpurun_out/br_$B.json 2>gpurun_out/br_$B.err
  python -c "import json; d=json.load(open('gpurun_out/br_$B.json')); print('branches=$B', round(d['value']), round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/br_$B.err
done
SFX_GRAPH_BRANCHES=1 timeout 300 python tools/layer_bench.py 2>&1 | tail -3
SFX_GRAPH_BRANCHES=0 timeout 300 python tools/layer_bench.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "program_api or encoder or deterministic or c5_full" 2>&1 | tail -2
