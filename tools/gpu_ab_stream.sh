# device-path cost of the host-streaming gate code (A/B per C5 group and C1/C2/C4)
for C in C5 C1 C2 C4; do timeout 300 python tools/ab_kernels.py $C default host_stream=1 default host_stream=1 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], d['group'], d['variant'], d['regs'], d['median_us'], d['gbs'])"; done
