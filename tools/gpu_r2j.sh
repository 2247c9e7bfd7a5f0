# round 2j: reciprocal for reduction-dependent divisors — full GPU suite, A/B against IEEE division (SFX_EXACT_DIV=1)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2j_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2j_pytest.log
timeout 600 python tools/long_rows_bench.py softmax > gpurun_out/r2j_longrows_rcp.jsonl 2>&1
SFX_EXACT_DIV=1 timeout 600 python tools/long_rows_bench.py softmax > gpurun_out/r2j_longrows_div.jsonl 2>&1
for i in 1 2; do
  for C in C2 C5; do
    timeout 600 python bench.py --config $C --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2j_${C}_rcp_$i.json 2>/dev/null
    SFX_EXACT_DIV=1 timeout 600 python bench.py --config $C --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2j_${C}_div_$i.json 2>/dev/null
  done
done
