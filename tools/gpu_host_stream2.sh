bash tools/gpu_ab_stream.sh
SFX_HOST_CHUNK_BYTES=4096 timeout 600 python tests/host_stream_check.py
for C in C5 C2 C1 C4; do python tools/e2e_probe.py $C 2>&1 | grep -v Warn; done
