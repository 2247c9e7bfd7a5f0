# literal tier (the reference's own blocks / arena / barriers) vs the templates, per group
for C in C1 C2 C3 C4 C5; do timeout 600 python tools/ab_kernels.py $C default strategy=literal 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('$C', d['group'], d['variant'], d['grid'], d['smem'], d['median_us'], d['gbs'])"; done
