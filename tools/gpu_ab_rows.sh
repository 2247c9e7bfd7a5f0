# row-template residency sweep on C5's rows (h1/h2: 768-wide rows, 3 streamed inputs; probs_d) and C1/C2
timeout 600 python tools/ab_kernels.py C5 default pipe_ctas_per_sm=8 pipe_ctas_per_sm=7 threads_per_row=32 2>&1 | grep -v Warn | grep -E '"group": "(h1|probs_d)"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['group'], d['variant'], d['regs'], d['grid'], d['median_us'], d['gbs'], d['vs_same_size_copy'])"
for C in C1 C2; do timeout 600 python tools/ab_kernels.py $C default pipe_ctas_per_sm=8 pipe_ctas_per_sm=6 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$C', d['group'], d['variant'], d['regs'], d['grid'], d['median_us'], d['gbs'], d['vs_same_size_copy'])"; done
