# round 2v: store-form A/B on the write-carrying column kernel (C3b db) and maps
mkdir -p gpurun_out
for X in none SFX_EXP_WB_STORES SFX_EXP_ST_NOCLOBBER; do
  if [ $X = none ]; then E=""; else E="SFX_EXPERIMENT=$X"; fi
  env $E timeout 600 python tools/ab_kernels.py C3b default items_per_thread=8 items_per_thread=24 > gpurun_out/r2v_C3b_$X.jsonl 2>> gpurun_out/r2v.err
  env $E timeout 600 python tools/ab_kernels.py C4 default > gpurun_out/r2v_C4_$X.jsonl 2>> gpurun_out/r2v.err
done
