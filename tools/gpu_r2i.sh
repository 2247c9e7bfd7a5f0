# round 2i: softmax statistics in one cluster combine (two local passes) — tests, A/B, ncu; C1 2-warp rows in flight
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "long or special or softmax or rows" > gpurun_out/r2i_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2i_pytest.log
timeout 900 python tools/long_rows_bench.py softmax > gpurun_out/r2i_longrows.jsonl 2> gpurun_out/r2i_longrows.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2i_rowcl_osm python tools/long_rows_bench.py softmax_1024 --variant='{}' > gpurun_out/r2i_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_rowcl" -s 3 -c 1 -o gpurun_out/r2i_rowcl_2lv python tools/long_rows_bench.py softmax_1024 --variant='{"row_pipeline": 4}' > gpurun_out/r2i_ncu2.log 2>&1
SIG=$(python -c "
import sys; sys.path.insert(0,'.')
import paper_1811_05213_b200 as P
g, rep, _ = P.load_bundle('workloads/plans/C1.full.json')
print(P.codegen(g, rep.kernels[0].program)[2].rsplit('sig=',1)[1].strip())")
printf "%s|0|64|0|0|12.72|13.30|C1/y test\n" "$SIG" > gpurun_out/r2i_tp64.txt
for i in 1 2; do
  timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_C1_default_$i.json 2>/dev/null
  SFX_TEMPLATE_PARAMS=gpurun_out/r2i_tp64.txt timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_C1_tpr64_$i.json 2>/dev/null
done
