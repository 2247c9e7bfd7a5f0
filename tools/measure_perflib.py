"""Measured B200 backend for the reference's performance library.

The paper's tuner looks schedules up in a performance library filled by
building, running and timing kernels (§4.4); the reference artifact
fills it with a synthetic cost model instead (tuning.cpp:169-201) and stores it
as text `opcode|shape|split_dim|sword|sched_type|block_threads|extra|cost_us|synthetic`
(tuning.cpp:41-125).  This tool times every fusion group of a plan bundle on
the B200 (CUDA events, median, inputs > L2) and writes non-synthetic entries
(`synthetic=0`) for the keys the reference plan used (make_perf_key,
tuning.cpp:154-167).  A fused group is one kernel, so its measured time is
split over the group's scheduled members in proportion to the reference's own
per-op estimate (bytes x expensive factor, tuning.cpp:169-190); summed back by
plan_cost_us (tuning.cpp:192-211) the plan costs exactly the measured time.
The reference's merge policy (non-synthetic wins) then lets `stitchfuse
perflib merge` / `compile_graph` consume it.

    python tools/measure_perflib.py C5 -o workloads/perflib/C5.b200.lib
"""

import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_05213_b200 import host as H  # noqa: E402

EXPENSIVE = H.EXPENSIVE  # default_expensive (ir.cpp:32-45)


def opcode_name(ins):  # ir.cpp opcode_name
    return ins.op


def perf_key(ins, sched, block_threads):  # make_perf_key, tuning.cpp:154-167
    split_dim, sword, stype = sched
    extra = str(block_threads // 32) if ins.op in ("reduce", "transpose") else "-"
    return "|".join([opcode_name(ins), ",".join(str(d) for d in ins.shape), str(split_dim), str(sword), stype,
                     str(block_threads), extra])


def est_weight(g, ins):  # estimate_cost_us numerator (occupancy is common to the plan)
    b = ins.numel() * 4 + sum(g.at(o).numel() * 4 for o in ins.operands)
    return b * (2.0 if ins.op in EXPENSIVE else 1.0)


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("-o", "--out", required=True)
    ap.add_argument("--size", default="full")
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    bundle_path = os.path.join(ROOT, "workloads", "plans", f"{args.config}.{args.size}.json")
    g, rep, bundle = H.load_bundle(bundle_path)
    ctx = H.Context(0)
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    lines = [f"# measured on {torch.cuda.get_device_name(dev)} by tools/measure_perflib.py "
             f"({args.config}.{args.size}); cost_us = median CUDA-event time of the group's single "
             "stitched launch, split over its scheduled members by the reference's per-op estimate"]
    for kb in bundle["kernels"]:
        prog = [k.program for k in rep.kernels if k.program.fusion_root == kb["fusion_root"]][0]
        k = H.Kernel(ctx, g, prog)
        ids = list(k.input_ids)
        per_set = sum(g.at(i).numel() * 4 for i in ids) + sum(g.at(r).numel() * 4 for r in prog.roots)
        nsets = max(1, min(8, math.ceil(3 * l2 / per_set)))
        sets = [([torch.rand(g.at(i).shape, device=dev) for i in ids],
                 [torch.empty(g.at(r).shape, device=dev) for r in prog.roots]) for _ in range(nsets)]
        s = torch.cuda.Stream(device=dev)
        for i in range(3):
            a, b = sets[i % nsets]
            k.launch([t.data_ptr() for t in a], [t.data_ptr() for t in b], s.cuda_stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for i in range(args.reps):
            a, b = sets[i % nsets]
            ev[i][0].record(s)
            k.launch([t.data_ptr() for t in a], [t.data_ptr() for t in b], s.cuda_stream)
            ev[i][1].record(s)
        torch.cuda.synchronize()
        us = sorted(x.elapsed_time(y) * 1e3 for x, y in ev)[args.reps // 2]
        sched = kb["per_instruction"]
        w = {m: est_weight(g, g.at(m)) for m in sched}
        tot = sum(w.values()) or 1.0
        for m, sc in sorted(sched.items()):
            cost = us * w[m] / tot
            lines.append(f"{perf_key(g.at(m), sc, kb['block_threads'])}|{cost:.9g}|0")
        print(f"{kb['fusion_root']}: {us:.2f} us over {len(sched)} scheduled member(s) [{k.info['entry']}]")
        k.close()
        del sets
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
