# register row template: variance folded in the mean's phase (SFX_ROW_VAR2=1) vs default, C1 and C5's LayerNorm groups
mkdir -p gpurun_out/r2bc
for i in 1 2 3; do
  timeout 600 python tools/ab_kernels.py C1 default >> gpurun_out/r2bc/ab_C1_default.jsonl 2>> gpurun_out/r2bc/ab.err
  SFX_ROW_VAR2=1 timeout 600 python tools/ab_kernels.py C1 default >> gpurun_out/r2bc/ab_C1_var2.jsonl 2>> gpurun_out/r2bc/ab.err
done
for i in 1 2; do
  timeout 600 python tools/ab_kernels.py C5 default >> gpurun_out/r2bc/ab_C5_default.jsonl 2>> gpurun_out/r2bc/ab.err
  SFX_ROW_VAR2=1 timeout 600 python tools/ab_kernels.py C5 default >> gpurun_out/r2bc/ab_C5_var2.jsonl 2>> gpurun_out/r2bc/ab.err
done
SFX_ROW_VAR2=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "configs_small or full_size or c5_full or long_and_odd or special_values or random_graphs or tma_row or resident or head_split" > gpurun_out/r2bc/pytest_var2.log 2>&1; echo rc=$? >> gpurun_out/r2bc/pytest_var2.log
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r2bc/C1_default.json 2>/dev/null
SFX_ROW_VAR2=1 timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r2bc/C1_var2.json 2>/dev/null
tail -2 gpurun_out/r2bc/pytest_var2.log
for f in gpurun_out/r2bc/ab_*.jsonl; do echo $f; cut -c1-220 $f; done
python -c "
import json
for n in ('C1_default','C1_var2'):
    d=json.load(open('gpurun_out/r2bc/'+n+'.json')); print(n, round(d['value']), d['roofline']['frac'], d['per_kernel'][0]['ms']*1000)
"
tail -5 gpurun_out/r2bc/ab.err
