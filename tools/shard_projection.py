"""Strong-scaling projection on ONE GPU (the box gpurun gives has one): for each
named config and n in {1, 2, 4, 8}, time one rank's batch shard (the reference's
own plan of the b/n shard graph, workloads/plans/<C>.shard<n>.json) alone, the
way bench.py times a rank (CUDA-graph replay, rotating input sets > 3x L2,
independent instances in flight: 4 below 512 MB, 2 above), and
project the n-GPU job as n x (shard bytes / shard time).  The projection assumes
ranks do not interfere (true on this path: no collective except C3's 4 KiB
column combine, which it leaves out) — an upper bound on bench.py --gpus n, and
the per-rank launch / ramp cost that small shards expose.

    python tools/shard_projection.py [C1 C5 ...]      # GPU box; one JSON line per (config, n)
"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1811_05213_b200 import host as H  # noqa: E402


def time_plan(ctx, path, steps=200, warmup=5):
    g, rep, _ = H.load_bundle(path)
    cg = H.CompiledGraph(ctx, g, rep)
    dev = torch.device("cuda", 0)
    per_set = sum(g.at(p).numel() * 4 for p in cg.param_ids) + sum(g.at(o).numel() * 4 for o in g.outputs)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    has_ws = any(k.info["workspace_bytes"] > 0 for k in cg.kernels)
    inflight = 4 if per_set <= (512 << 20) else 2 if per_set <= (16 << 30) else 1  # as bench.py (one rank: no peers)
    if os.environ.get("PROJ_INFLIGHT"):  # A/B: instances in flight
        inflight = int(os.environ["PROJ_INFLIGHT"])
    nsets = max(inflight, min(64, math.ceil(3 * l2 / per_set)))
    sets = []
    for _ in range(nsets):
        ins = [torch.rand(g.at(p).shape, device=dev) * 2 - 1 for p in cg.param_ids]
        outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
        sets.append(([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], ins, outs))
    streams = [torch.cuda.Stream(device=dev) for _ in range(inflight)]
    torch.cuda.synchronize()

    def step(i):
        pi, po, _, _ = sets[i % nsets]
        cg.run(pi, po, stream=streams[i % inflight].cuda_stream, cuda_graph=True)

    for i in range(max(warmup * inflight, 2 * nsets)):  # every buffer set's CUDA graph captured before timing
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = streams[0]
    e0.record(main)
    for s in streams[1:]:
        s.wait_event(e0)
    for i in range(steps):
        step(i)
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    algo = sum(k.info["algorithmic_bytes"] for k in cg.kernels)
    launches = len(cg.kernels) + len(cg.barrier_kernels)
    cg.close()
    return ms, algo, inflight, launches


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C4b", "C4t", "C5"]
    ctx = H.Context(0)
    for name in names:
        base = None
        for n in (1, 2, 4, 8):
            path = os.path.join(ROOT, "workloads", "plans", f"{name}.full.json" if n == 1 else f"{name}.shard{n}.json")
            ms, algo, inflight, launches = time_plan(ctx, path)
            gbs_rank = algo / (ms * 1e-3) / 1e9
            proj = n * gbs_rank
            if base is None:
                base = proj
            print(json.dumps({"config": name, "n": n, "plan": os.path.basename(path), "rank_bytes": algo,
                              "rank_ms": round(ms, 4), "rank_gbs": round(gbs_rank, 1), "instances_in_flight": inflight,
                              "launches_per_graph": launches, "projected_job_gbs": round(proj, 1),
                              "projected_efficiency": round(proj / (n * base), 3)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
