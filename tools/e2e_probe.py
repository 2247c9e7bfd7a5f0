"""Host-path (sfx_graph_run_host) timing of one config, pinned buffers; env
SFX_HOST_STREAM / SFX_HOST_CHUNK_BYTES select the schedule."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
g, rep, _ = H.load_bundle(os.path.join(ROOT, "workloads", "plans", f"{cfg}.full.json"))
ctx = H.Context(0)
cg = H.CompiledGraph(ctx, g, rep)
pin_in = [torch.rand(g.at(p).shape).pin_memory() for p in cg.param_ids]
pin_out = [torch.empty(g.at(o).shape).pin_memory() for o in g.outputs]
ai = (C.c_void_p * len(pin_in))(*[t.data_ptr() for t in pin_in])
ao = (C.c_void_p * len(pin_out))(*[t.data_ptr() for t in pin_out])
s = torch.cuda.Stream()
ts = []
for i in range(6):
    t = time.perf_counter()
    H._check(H.lib().sfx_graph_run_host(cg.h, ai, len(pin_in), ao, len(pin_out), C.c_void_p(s.cuda_stream)))
    ts.append(time.perf_counter() - t)
b = sum(t.numel() * 4 for t in pin_in + pin_out)
m = min(ts[1:])
print(cfg, os.environ.get("SFX_HOST_STREAM", "1"), os.environ.get("SFX_HOST_CHUNK_BYTES", "16M"),
      f"{m * 1e3:.2f} ms  {b / m / 1e9:.1f} GB/s", flush=True)
