mkdir -p gpurun_out
timeout 2400 oracle/_ref/device_parity random 43000 200 --fuse-dot-alternate --literal > gpurun_out/r2ai_packed.log 2>&1; echo rc=$? >> gpurun_out/r2ai_packed.log
SFX_DOT_PACKED=0 timeout 2400 oracle/_ref/device_parity random 43000 200 --fuse-dot-alternate --literal > gpurun_out/r2ai_fmul.log 2>&1; echo rc=$? >> gpurun_out/r2ai_fmul.log
timeout 2400 oracle/_ref/device_parity random 43000 200 --fuse-dot-alternate > gpurun_out/r2ai_auto.log 2>&1; echo rc=$? >> gpurun_out/r2ai_auto.log
