"""Batch-norm at the bench shapes (colbc template): the one-pass second moment
(default) and the two-level form (SFX_COLBC_TWO_PASS=1, run in a child process:
the lowering reads the variable once per compiled kernel) against the fp64 and
fp32 oracles, element by element (tests' strict tolerance), and against each
other.  The offset case (x = 1000 + 0.01 u) is ill-conditioned in fp32: d = x - mean
carries ~ulp(1000) of the input's own rounding, so any fp32 evaluation of the graph
differs from the fp64 oracle there; it checks that the shifted sums do not add
cancellation error beyond the two-level form's."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
import sfx_testlib as T  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402
from workloads import configs  # noqa: E402
from make_extra_plans import bn_graph  # noqa: E402

CASES = {"batchnorm_65536x256": bn_graph([65536, 256], [0]),
         "batchnorm_nhwc_64x56x56x256": bn_graph([64, 56, 56, 256], [0, 1, 2]),
         "batchnorm_offset_65536x256": bn_graph([65536, 256], [0]),
         "batchnorm_nchw_64x256x56x56": bn_graph([64, 256, 56, 56], [0, 2, 3]),
         "batchnorm_nchw_32x64x112x112": bn_graph([32, 64, 112, 112], [0, 2, 3])}
OUT = os.path.join(tempfile.gettempdir(), "colbc_check")
os.makedirs(OUT, exist_ok=True)


def load(name):
    bpath = os.path.join(OUT, name + ".plan.json")
    if not os.path.exists(bpath):
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            f.write(configs.dumps(CASES[name]))
        out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_tool"), "plan", f.name], check=True,
                             capture_output=True, text=True).stdout
        open(bpath, "w").write(out)
    g, rep, _ = H.load_bundle(bpath)
    inputs = T.gen_inputs_fast(g, 5, -1.0, 1.0)
    if "offset" in name:
        inputs["x"] = (inputs["x"] * np.float32(0.01) + np.float32(1000.0)).astype(np.float32)
    return g, rep, inputs


def run_device(mode):
    import torch
    ctx = H.Context(0)
    dev = torch.device("cuda", 0)
    for name in CASES:
        g, rep, inputs = load(name)
        prog = rep.kernels[-1].program
        k = H.Kernel(ctx, g, prog)
        ins = [torch.from_numpy(np.ascontiguousarray(inputs[i])).to(dev) for i in k.input_ids]
        outs = [torch.empty(g.at(r).shape, device=dev) for r in prog.roots]
        k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs])
        torch.cuda.synchronize()
        np.save(os.path.join(OUT, f"{name}.{mode}.npy"), outs[0].cpu().numpy())
        k.close()


if len(sys.argv) > 1 and sys.argv[1] == "--device":
    run_device(sys.argv[2])
    sys.exit(0)
for mode, env in (("one_pass", "0"), ("two_pass", "1")):
    subprocess.run([sys.executable, __file__, "--device", mode], check=True, env=dict(os.environ, SFX_COLBC_TWO_PASS=env))
ok = True
for name in CASES:
    g, rep, inputs = load(name)
    ref64 = T.interpret(g, inputs, 1)["y"].astype(np.float64)
    ref32 = T.interpret(g, inputs, 0)["y"].astype(np.float64)
    ys = {m: np.load(os.path.join(OUT, f"{name}.{m}.npy")) for m in ("one_pass", "two_pass")}
    for m, y in ys.items():
        y64 = y.astype(np.float64)
        good = T.strict_close(y, ref64.astype(np.float32))
        if "offset" not in name:
            ok &= good
        print(json.dumps({"case": name, "mode": m, "strict_close_fp64_oracle": good,
                          "max_abs_vs_fp64": float(np.abs(y64 - ref64).max()),
                          "max_abs_vs_fp32_oracle": float(np.abs(y64 - ref32).max())}), flush=True)
    d = np.abs(ys["one_pass"].astype(np.float64) - ys["two_pass"].astype(np.float64))
    print(json.dumps({"case": name, "one_vs_two_max_abs": float(d.max()),
                      "identical_fraction": float((ys["one_pass"] == ys["two_pass"]).mean())}), flush=True)
sys.exit(0 if ok else 1)
