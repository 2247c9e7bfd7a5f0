# round 2t: C1 finer row granularity — single-launch A/B and the benchmark value (instances in flight)
mkdir -p gpurun_out
SIG=sfx_row-0d0a6822502c737d
printf "%s|1|128|0|0|0|0|test\n" "$SIG" > gpurun_out/r2t_tp_128x1.txt
printf "%s|1|256|0|0|0|0|test\n" "$SIG" > gpurun_out/r2t_tp_256x1.txt
printf "%s|2|64|0|0|0|0|test\n" "$SIG" > gpurun_out/r2t_tp_64x2.txt
timeout 600 python tools/ab_kernels.py C1 default threads_per_row=128,rows_per_cta=1 threads_per_row=256,rows_per_cta=1 threads_per_row=64,rows_per_cta=2 > gpurun_out/r2t_ab_C1.jsonl 2> gpurun_out/r2t_ab.err
for i in 1 2 3; do
  timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2t_C1_default_$i.json 2>/dev/null
  for v in 128x1 256x1 64x2; do
    SFX_TEMPLATE_PARAMS=gpurun_out/r2t_tp_$v.txt timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2t_C1_${v}_$i.json 2>/dev/null
  done
done
