# round 2p: new parity shapes (masked long softmax with a cached member feeding two roots; two-input colbc ring)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "long_and_odd or special_rows or peer" > gpurun_out/r2p_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2p_pytest.log
for TOOL in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 python tools/sanitize_check.py none > gpurun_out/r2p_sanitize_$TOOL.log 2>&1; echo "$TOOL rc=$?" >> gpurun_out/r2p_sanitize.txt
done
