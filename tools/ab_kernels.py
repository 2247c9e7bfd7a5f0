"""A/B timing of lowering variants for one workload's groups (GPU box).

    python tools/ab_kernels.py C1 row_pipeline=1 row_pipeline=2

Each variant: compile every group with those options, check the group's roots
against the oracle on a deterministic input (strict tolerance, fp64 oracle for
reduce-dependent roots), then time each kernel alone with CUDA events over
rotating buffer sets (> 3x L2).  Prints one JSON line per (variant, group).
"""

import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import sfx_testlib as T  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402


def parse(kv):
    out = {}
    for a in kv:
        k, v = a.split("=")
        out[k] = v if k == "strategy" else int(v)
    return out


def main():
    cfg = sys.argv[1]
    variants = [parse(v.split(",")) if v != "default" else {} for v in sys.argv[2:]] or [{}]
    size = os.environ.get("AB_SIZE", "full")
    g, rep, _ = H.load_bundle(os.path.join(ROOT, "workloads", "plans", f"{cfg}.{size}.json"))
    ctx = H.Context(0)
    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for var in variants:
        for kp in rep.kernels:
            k = H.Kernel(ctx, g, kp.program, **var)
            ids = list(k.input_ids)
            per_set = sum(g.at(i).numel() * 4 for i in ids) + sum(g.at(r).numel() * 4 for r in kp.program.roots)
            nsets = max(1, min(8, math.ceil(3 * l2 / per_set)))
            # correctness on set 0 (deterministic stream) vs the oracle
            sub_inputs = {}
            if per_set < 2 ** 31:
                full_in = T.gen_inputs_fast(g, 5, -1.0, 1.0) if size == "small" else None
            sets = []
            for s in range(nsets):
                ins = [torch.rand(g.at(i).shape, device=dev) * 2 - 1 for i in ids]
                outs = [torch.empty(g.at(r).shape, device=dev) for r in kp.program.roots]
                sets.append((ins, outs))
            ok = None
            if size == "small":
                ins = [torch.from_numpy(full_in[i]).to(dev) if i in full_in else sets[0][0][n]
                       for n, i in enumerate(ids)]
                k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in sets[0][1]])
                torch.cuda.synchronize()
                ref = T.interpret(g, full_in, 1)
                ok = all(T.strict_close(o.cpu().numpy(), ref[r]) for o, r in zip(sets[0][1], kp.program.roots))
            s = torch.cuda.Stream(device=dev)
            reps = 30
            for i in range(5):
                ins, outs = sets[i % nsets]
                k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for i in range(reps):
                ins, outs = sets[i % nsets]
                ev[i][0].record(s)
                k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
                ev[i][1].record(s)
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in ev)
            med = ms[len(ms) // 2]
            # back to back (PDL-chained launches, as in bench.py's per-kernel figure)
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(s)
            for i in range(reps):
                ins, outs = sets[i % nsets]
                k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
            b1.record(s)
            torch.cuda.synchronize()
            b2b = b0.elapsed_time(b1) / reps
            gbs = k.info["algorithmic_bytes"] / (med * 1e-3) / 1e9
            # same-size copy (torch copy_ of half the algorithmic bytes each way),
            # the achievable single-launch bandwidth at this size
            half = k.info["algorithmic_bytes"] // 8
            cps = [(torch.empty(half, device=dev), torch.empty(half, device=dev)) for _ in range(nsets)]
            for i in range(3):
                cps[i % nsets][1].copy_(cps[i % nsets][0])
            cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            cs = torch.cuda.current_stream()
            for i in range(reps):
                cev[i][0].record(cs)
                cps[i % nsets][1].copy_(cps[i % nsets][0])
                cev[i][1].record(cs)
            torch.cuda.synchronize()
            cmed = sorted(a.elapsed_time(b) for a, b in cev)[reps // 2]
            del cps
            print(json.dumps({"config": cfg, "variant": var, "group": kp.program.fusion_root,
                              "kernel": k.info["entry"], "regs": k.info["registers"], "grid": k.info["grid"],
                              "smem": k.info["smem_bytes"], "median_us": round(med * 1e3, 2),
                              "b2b_us": round(b2b * 1e3, 2),
                              "b2b_frac": round(k.info["algorithmic_bytes"] / (b2b * 1e-3) / 1e9 / peak, 3),
                              "gbs": round(gbs), "frac": round(gbs / peak, 3),
                              "same_size_copy_us": round(cmed * 1e3, 2),
                              "vs_same_size_copy": round(cmed / med, 3), "parity_ok": ok}), flush=True)
            k.close()
            del sets


if __name__ == "__main__":
    main()
