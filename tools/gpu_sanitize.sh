# compute-sanitizer over the stitched kernels of every small config (both tiers)
# and 12 reference random graphs; summaries into gpurun_out/sanitize_*.log
for TOOL in memcheck racecheck synccheck initcheck; do
  SFX_SANITIZER=$TOOL timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 python tools/sanitize_check.py > gpurun_out/sanitize_$TOOL.log 2>&1
  echo "$TOOL rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitize_$TOOL.log | sort | uniq -c | head -5
done
