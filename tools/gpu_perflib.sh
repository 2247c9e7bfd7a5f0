mkdir -p gpurun_out/perflib
for C in C1 C2 C3 C4 C5; do timeout 300 python tools/measure_perflib.py $C -o gpurun_out/perflib/$C.b200.lib 2>&1 | tail -6; done
ncu --set full --clock-control none --import-source on -k regex:"sfx_(row_probs_d|map_gelu|row_h1|map_ctx_r)" -s 4 -c 4 -o gpurun_out/r01b_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/
