# one-pass second moments in the colbc template: parity (tests + bench shapes vs the fp64 oracle), A/B timing, ncu, sanitizers
mkdir -p gpurun_out/r2aw
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bn or colbc or long_and_odd or peer or sync" > gpurun_out/r2aw/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2aw/pytest.log
timeout 600 python tools/colbc_check.py > gpurun_out/r2aw/check.jsonl 2> gpurun_out/r2aw/check.err; echo check rc=$?
timeout 600 python tools/long_rows_bench.py batchnorm --variant='{}' > gpurun_out/r2aw/one_pass.jsonl 2>&1
SFX_COLBC_TWO_PASS=1 timeout 600 python tools/long_rows_bench.py batchnorm --variant='{}' > gpurun_out/r2aw/two_pass.jsonl 2>&1
timeout 600 python tools/long_rows_bench.py batchnorm > gpurun_out/r2aw/variants.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2aw/colbc_65536 python tools/long_rows_bench.py batchnorm_65536 --variant='{}' > gpurun_out/r2aw/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_colbc" -s 3 -c 1 -o gpurun_out/r2aw/colbc_nhwc python tools/long_rows_bench.py batchnorm_nhwc --variant='{}' >> gpurun_out/r2aw/ncu.log 2>&1
for TOOL in memcheck racecheck synccheck; do
  SFX_SANITIZER=$TOOL timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 python tools/sanitize_check.py > gpurun_out/r2aw/sanitize_$TOOL.log 2>&1
  echo "$TOOL rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r2aw/sanitize_$TOOL.log | sort | uniq -c | head -3
done
tail -2 gpurun_out/r2aw/pytest.log; cat gpurun_out/r2aw/check.jsonl; cat gpurun_out/r2aw/one_pass.jsonl gpurun_out/r2aw/two_pass.jsonl
