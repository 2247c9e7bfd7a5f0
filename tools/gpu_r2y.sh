# round 2y: C1 shard plans (strong-scaling shards b/2, b/4, b/8 rows): default rows vs 4-warp rows per CTA
mkdir -p gpurun_out
for S in shard2 shard4 shard8; do
  AB_SIZE=$S timeout 600 python tools/ab_kernels.py C1 threads_per_row=32 threads_per_row=128,rows_per_cta=1 threads_per_row=64,rows_per_cta=1 > gpurun_out/r2y_C1_$S.jsonl 2>> gpurun_out/r2y.err
done
for S in shard2 shard4 shard8; do
  python -c "
import sys; sys.path.insert(0,'.')
import paper_1811_05213_b200 as P
g, rep, _ = P.load_bundle('workloads/plans/C1.$S.json')
print('$S', P.codegen(g, rep.kernels[0].program)[2].rsplit('sig=',1)[1].strip())" >> gpurun_out/r2y_sigs.txt
done
