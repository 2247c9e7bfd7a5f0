"""Throughput of the templates for long rows (rows beyond 1024 threads x 64
elements: softmax / LayerNorm with 128K-262K-wide rows) and for batch-norm
statistics broadcast back (colbc), planned by the
reference's compile_graph (oracle/_ref/ref_tool) at run time, timed with CUDA
events over rotating buffers (> L2), GB/s of compulsory bytes."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402
from workloads import configs  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_extra_plans import bn_graph  # noqa: E402

ONLY = [a for a in sys.argv[1:] if not a.startswith("--")]
CASES = {"batchnorm_65536x256": bn_graph([65536, 256], [0]),
         "batchnorm_262144x1024": bn_graph([262144, 1024], [0]),
         "batchnorm_nhwc_64x56x56x256": bn_graph([64, 56, 56, 256], [0, 1, 2]),
         "batchnorm_nchw_64x256x56x56": bn_graph([64, 256, 56, 56], [0, 2, 3]),
         "batchnorm_nchw_32x64x112x112": bn_graph([32, 64, 112, 112], [0, 2, 3]),
         "softmax_1024x131072": configs.c2_softmax(B=1, H=1, S=1024, L=131072),
         "layernorm_1024x131072": configs.c1_layernorm(R=1024, C=131072),
         "softmax_256x262144": configs.c2_softmax(B=1, H=1, S=256, L=262144)}
dev = torch.device("cuda", 0)
ctx = H.Context(0)
for name, doc in CASES.items():
    if ONLY and not any(name.startswith(o) for o in ONLY):
        continue
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(configs.dumps(doc))
        path = f.name
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_tool"), "plan", path], check=True,
                         capture_output=True, text=True).stdout
    os.unlink(path)
    bpath = os.path.join(tempfile.gettempdir(), name + ".json")
    open(bpath, "w").write(out)
    g, rep, b = H.load_bundle(bpath)
    variants = [{}] + ([{"items_per_thread": 4}, {"items_per_thread": 16}, {"pipe_ctas_per_sm": 3}, {"pipe_ctas_per_sm": 4}] if "nchw" in name else [{"row_pipeline": 1}, {"items_per_thread": 4}, {"items_per_thread": 2}, {"pipe_ctas_per_sm": 1}, {"pipe_ctas_per_sm": 3}] if name.startswith("batchnorm") else [{"row_pipeline": 1}, {"pipe_stages": 8}, {"row_pipeline": 5}, {"row_pipeline": 3}])
    if "--literal" in sys.argv:
        variants.append({"strategy": "literal"})
    pick = [a[len("--variant="):] for a in sys.argv if a.startswith("--variant=")]
    if pick:  # one variant only (e.g. for an ncu capture): --variant='{"row_pipeline": 4}'
        variants = [json.loads(pick[0])]
    for kw in variants:
        k = H.Kernel(ctx, g, rep.kernels[0].program, **kw)
        ids = list(k.input_ids)
        sets = [([torch.rand(g.at(i).shape, device=dev) * 2 - 1 for i in ids],
                 [torch.empty(g.at(r).shape, device=dev) for r in rep.kernels[0].program.roots]) for _ in range(2)]
        reps = 10 if kw else 30
        for i in range(3):
            k.launch([t.data_ptr() for t in sets[i % 2][0]], [t.data_ptr() for t in sets[i % 2][1]])
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i, (a, e) in enumerate(ev):
            a.record()
            k.launch([t.data_ptr() for t in sets[i % 2][0]], [t.data_ptr() for t in sets[i % 2][1]])
            e.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(e) for a, e in ev)[reps // 2]
        print(json.dumps({"case": name, "variant": kw, "strategy": k.info["strategy"], "regs": k.info["registers"],
                          "us": round(ms * 1e3, 1), "gbs": round(k.info["algorithmic_bytes"] / ms / 1e6)}), flush=True)
        k.close()
        del sets
