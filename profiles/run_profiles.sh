#!/bin/bash
# The exact profiling commands behind profiles/<tag>_*.md (run on the GPU box
# through gpurun; results come back in gpurun_out/ and are summarised here by
# profiles/ncu_summary.py).  Never a bench number: ncu serialises and replays.
set -x
TAG=${1:-r01}
# 1) launch list of the benchmark command (per-launch device time, cold cache)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# 2) full capture of the C5 groups' kernels (one launch each after warm-up)
ncu --set full --clock-control none --import-source on \
    -k regex:"sfx_(row_probs_d|map_gelu|row_h1|row_h2|map_ctx_r)" -s 5 -c 5 \
    -o gpurun_out/${TAG}_C5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
# 3) full capture of the single-group configs (C3b: both groups; C4t: the smem-tiled transpose)
for C in C1 C2 C3 C3b C4 C4b C4t; do
  N=1; [ $C = C3b ] && N=2
  ncu --set full --clock-control none --import-source on -k regex:"sfx_" -s $((2*N)) -c $N \
      -o gpurun_out/${TAG}_${C} python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
