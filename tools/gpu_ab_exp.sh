# prelude experiment A/B: evict-first streaming loads
for E in NONE SFX_LD_EF NONE SFX_LD_EF; do
  if [ $E = NONE ]; then unset SFX_EXPERIMENT; else export SFX_EXPERIMENT=$E; fi
  for C in C5 C2 C3 C4; do timeout 300 python tools/ab_kernels.py $C default 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$E', '$C', d['group'], d['median_us'], d['gbs'])"; done
done
