# full GPU suite + per-config benches (same as gpu_check.sh) + e2e probe
bash tools/gpu_check.sh
for C in C5 C2 C1; do python tools/e2e_probe.py $C 2>&1 | grep -v Warn; done
