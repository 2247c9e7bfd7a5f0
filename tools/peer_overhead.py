"""Cost of the in-kernel cross-rank combine (cross_rank=1) measured on one GPU:
a peer group of one rank runs the whole protocol (partials pushed to the
arena, release flag, acquire wait, rank-ordered fold) against itself.  Times
the C3 column kernel with and without it (CUDA events, rotating buffers)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
g, rep, _ = H.load_bundle(os.path.join(ROOT, "workloads", "plans", f"{cfg}.full.json"))
dev = torch.device("cuda", 0)
res = {}
for mode in ("plain", "peer"):
    ctx = H.Context(0)
    if mode == "peer":
        ctx.peer_init(0, 1, lambda h: [h])
    cg = H.CompiledGraph(ctx, g, rep, cross_rank=int(mode == "peer"))
    sets = []
    for _ in range(3):
        ins = [torch.rand(g.at(p).shape, device=dev) * 2 - 1 for p in cg.param_ids]
        outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
        sets.append((ins, outs))
    s = torch.cuda.Stream()
    for i in range(10):
        ins, outs = sets[i % 3]
        cg.run([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], stream=s.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for i, (a, b) in enumerate(ev):
        ins, outs = sets[i % 3]
        a.record(s)
        cg.run([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], stream=s.cuda_stream)
        b.record(s)
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    res[mode] = {"median_us": round(ms[25] * 1e3, 2), "db_sum": float(sets[0][1][0].double().sum())}
    cg.close()
    ctx.close()
res["overhead_us"] = round(res["peer"]["median_us"] - res["plain"]["median_us"], 2)
print(json.dumps({"config": cfg, **res}))
