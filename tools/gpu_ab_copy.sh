for C in C1 C2 C3 C4 C4b C5; do timeout 600 python tools/ab_kernels.py $C default 2>&1 | grep '^{'; done
