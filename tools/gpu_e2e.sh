for C in C5 C2 C1; do
SFX_HOST_STREAM=0 python tools/e2e_probe.py $C
python tools/e2e_probe.py $C
SFX_HOST_CHUNK_BYTES=4194304 python tools/e2e_probe.py $C
SFX_HOST_CHUNK_BYTES=67108864 python tools/e2e_probe.py $C
SFX_HOST_CHUNK_BYTES=8388608 python tools/e2e_probe.py $C
done
