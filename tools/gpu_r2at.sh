# column-workspace kernels with instances in flight (per-stream workspaces): C3 / C3b bench lines, concurrency test, projection for C3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "concurrent" > gpurun_out/r2at_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2at_pytest.log
for C in C3 C3b; do for i in 1 2; do timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2at_${C}_$i.json 2>> gpurun_out/r2at.err; done; done
for C in C3 C3b; do timeout 600 python bench.py --config $C --no-cpu-baseline --inflight 1 > gpurun_out/r2at_${C}_if1.json 2>> gpurun_out/r2at.err; done
timeout 900 python tools/shard_projection.py C3 > gpurun_out/r2at_proj.jsonl 2>> gpurun_out/r2at.err
