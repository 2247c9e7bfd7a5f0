"""Whole BERT-base encoder layer (C5L: C5's non-MatMul groups chained through
the matmul barriers, reference plan in workloads/plans/C5L.full.json) on one
B200: CUDA-graph replay of the compiled module, per-kernel CUDA-event times,
and the split between the stitched groups (HBM-bound, GB/s) and the matmul
kernels (SIMT fp32, TFLOP/s).  Inputs U(-1,1) resident in HBM.

    python tools/layer_bench.py [--steps 10] [--config C5L]
Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_05213_b200 import host as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5L")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = H.Context(0)
    g, rep, b = H.load_bundle(os.path.join(ROOT, "workloads", "plans", f"{args.config}.full.json"))
    cg = H.CompiledGraph(ctx, g, rep)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    ins = [torch.rand(g.at(p).shape, generator=gen, device=dev) * 2 - 1 for p in cg.param_ids]
    outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
    pi, po = [t.data_ptr() for t in ins], [t.data_ptr() for t in outs]
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        for _ in range(args.warmup):
            cg.run(pi, po, stream=s.cuda_stream, cuda_graph=True)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        before = ctx.launch_count()
        e0.record(s)
        for _ in range(args.steps):
            cg.run(pi, po, stream=s.cuda_stream, cuda_graph=True)
        e1.record(s)
        s.synchronize()
        launched = (ctx.launch_count() - before) // args.steps
        ms = e0.elapsed_time(e1) / args.steps
        assert torch.isfinite(outs[0]).all()

    # per-kernel times: each kernel alone on its own (device-resident) operands
    kernels = [(k, "group") for k in cg.kernels] + [(k, "unfused") for k in cg.barrier_kernels]
    scratch = {}

    def buf(node):
        if node in cg.param_ids:
            return ins[cg.param_ids.index(node)].data_ptr()
        if node not in scratch:
            scratch[node] = torch.empty(g.at(node).shape, device=dev)
        return scratch[node].data_ptr()

    from bench import Clocks  # nvidia-smi sampler (clocks under load)
    clocks = Clocks(0).start()
    rows = []
    for k, kind in kernels:
        out_ids = k.roots
        ip = [buf(i) for i in k.input_ids]
        op = [buf(o) for o in out_ids]
        reps = 40 if k.info["strategy"] == "dot" else 5  # matmuls: >= 100 ms, several clock samples
        with torch.cuda.stream(s):
            for _ in range(2):
                k.launch(ip, op, stream=s.cuda_stream)
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(s)
            for _ in range(reps):
                k.launch(ip, op, stream=s.cuda_stream)
            z.record(s)
            s.synchronize()
            t1 = time.perf_counter()
        t = a.elapsed_time(z) / reps
        row = {"kernel": k.info["entry"], "kind": kind, "strategy": k.info["strategy"], "ms": round(t, 4)}
        if k.info["strategy"] == "dot":
            node = g.at(out_ids[0])
            K = g.at(node.operands[0]).shape[-1]
            row["tflops"] = round(2.0 * node.numel() * K / t / 1e9, 2)
            # the SIMT ceiling at the clock the matmul actually ran at: 148 SMs x 128
            # FP32 lanes, one FMUL + one FADD per multiply-add (2 flops / 2 issues)
            ck = clocks.summary(t0, t1)
            row["clocks"] = ck
            if ck.get("sm_mhz"):
                ceil = 148 * 128 * ck["sm_mhz"] * 1e6 / 1e12
                row["simt_ceiling_tflops_at_clock"] = round(ceil, 2)
                row["frac_of_ceiling_at_clock"] = round(row["tflops"] / ceil, 3)
        else:
            row["gbs"] = round(k.info["algorithmic_bytes"] / t / 1e6, 1)
        rows.append(row)
    dot_ms = sum(r["ms"] for r in rows if r["strategy"] == "dot")
    other_ms = sum(r["ms"] for r in rows if r["strategy"] != "dot")
    clocks.stop()
    print(json.dumps({"config": args.config, "layer_ms": round(ms, 3), "launches_per_layer": launched,
                      "sum_kernel_ms": round(dot_ms + other_ms, 3), "matmul_ms": round(dot_ms, 3),
                      "non_matmul_ms": round(other_ms, 3), "kernels": rows}), flush=True)
    cg.close()
    ctx.close()


if __name__ == "__main__":
    main()
