"""Template parameter autotuner (GPU box): for every group of the committed
workload plans, time candidate template parameters against the defaults and
write the winners to the template parameter cache (PerfLibrary-style text,
see csrc/lower.cpp "template parameter cache").

    python tools/autotune.py [out_file] [configs...]

A candidate must beat the defaults by >= 2% (back-to-back launch average over
rotating buffer sets > 3x L2) and reproduce the default kernel's outputs
(strict tolerance; sums may differ in the last bits by summation order)."""

import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import sfx_testlib as T  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402

CANDIDATES = {
    "map": [dict(items_per_thread=u) for u in (1, 2, 4, 8)],
    "row": [dict(threads_per_row=t) for t in (32, 64, 128, 256)] + [dict(rows_per_cta=r) for r in (1, 2, 4)]
           + [dict(threads_per_row=t, rows_per_cta=r) for t in (64, 128) for r in (1, 4)],
    "col": [dict(pipe_ctas_per_sm=m, items_per_thread=u) for m, u in ((1, 24), (1, 32), (2, 8), (3, 12))],
}


def timed(k, g, prog, sets, reps=20):
    s = torch.cuda.Stream()
    def go(i):
        ins, outs = sets[i % len(sets)]
        k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], s.cuda_stream)
    for i in range(3):
        go(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record(s)
        for i in range(reps):
            go(i)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


def timed_inflight(k, sets, n=4, reps=40):
    """Per-launch time with n independent instances in flight (the benchmark's
    mode for graphs < 512 MB): round-robin over n streams and buffer sets."""
    ss = [torch.cuda.Stream() for _ in range(n)]
    def go(i):
        ins, outs = sets[i % len(sets)]
        k.launch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], ss[i % n].cuda_stream)
    for i in range(2 * n):
        go(i)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ss[0])
        for s in ss[1:]:
            s.wait_event(e0)
        for i in range(reps):
            go(i)
        for s in ss[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            ss[0].wait_event(ev)
        e1.record(ss[0])
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "template_params.txt")
    configs = sys.argv[2:] or ["C1", "C2", "C3", "C3b", "C4", "C4b", "C4t", "C5"]
    os.environ["SFX_TEMPLATE_PARAMS"] = "0"  # measure against the plain defaults
    ctx = H.Context(0)
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    lines = ["# template parameter cache: signature|rows_per_cta|threads_per_row|items_per_thread|"
             "pipe_ctas_per_sm|tuned_us|default_us|source",
             "# written by tools/autotune.py on one B200 (back-to-back launch averages, rotating buffer sets > 3x L2)"]
    done = set()
    for cfg in configs:
        g, rep, _ = H.load_bundle(os.path.join(ROOT, "workloads", "plans", f"{cfg}.full.json"))
        for kp in rep.kernels:
            prog = kp.program
            _, _, note = H.codegen(g, prog)
            strategy = note.split()[0]
            sig = note.rsplit("sig=", 1)[1].strip()
            if strategy not in CANDIDATES or sig in done:  # same group structure (C5 h1 / h2): measured once
                continue
            done.add(sig)
            base = H.Kernel(ctx, g, prog)
            ids = list(base.input_ids)
            per_set = sum(g.at(i).numel() * 4 for i in ids) + sum(g.at(r).numel() * 4 for r in prog.roots)
            nsets = max(1, min(6, math.ceil(3 * l2 / per_set)))
            gen = torch.Generator(device=dev)
            gen.manual_seed(7)
            sets = [([torch.rand(g.at(i).shape, generator=gen, device=dev) * 2 - 1 for i in ids],
                     [torch.empty(g.at(r).shape, device=dev) for r in prog.roots]) for _ in range(nsets)]
            t0 = timed(base, g, prog, sets)
            ref = [o.clone() for o in sets[0][1]]
            best = (t0, None)
            for kw in CANDIDATES[strategy]:
                try:
                    k = H.Kernel(ctx, g, prog, **kw)
                except H.ExecError:
                    continue
                t = timed(k, g, prog, sets)
                same = all(T.strict_close(o.cpu().numpy(), r.cpu().numpy()) for o, r in zip(sets[0][1], ref))
                k.close()
                print(cfg, prog.fusion_root, strategy, kw, round(t, 2), "default", round(t0, 2), "ok" if same else "MISMATCH",
                      flush=True)
                if same and t < best[0]:
                    best = (t, kw)
            # small groups run with instances in flight in the benchmark: the
            # winner must win there too, by >= 1% in this short burst (a kernel
            # that is faster alone can draw more power and lose under the
            # sustained power cap: C1 at 4 warps per row ties here, 10.34 vs
            # 10.40 us, and loses 3% of the benchmark value at an SM clock
            # 100 MHz lower, profiles/README.md)
            if best[1] is not None and per_set < (512 << 20) and len(sets) >= 4:
                k = H.Kernel(ctx, g, prog, **best[1])
                ti_best, ti_base = timed_inflight(k, sets), timed_inflight(base, sets)
                k.close()
                print(cfg, prog.fusion_root, "in flight", best[1], round(ti_best, 2), "default", round(ti_base, 2),
                      flush=True)
                if ti_best > 0.99 * ti_base:
                    best = (t0, None)
            base.close()
            if best[1] is not None and best[0] < 0.98 * t0:
                kw = best[1]
                lines.append("|".join([sig, str(kw.get("rows_per_cta", 0)), str(kw.get("threads_per_row", 0)),
                                       str(kw.get("items_per_thread", 0)), str(kw.get("pipe_ctas_per_sm", 0)),
                                       f"{best[0]:.2f}", f"{t0:.2f}", f"{cfg}/{prog.fusion_root}"]))
            else:  # measured, defaults kept (a hit: the group is not re-measured on miss)
                lines.append("|".join([sig, "0", "0", "0", "0", f"{t0:.2f}", f"{t0:.2f}",
                                       f"{cfg}/{prog.fusion_root} defaults kept"]))
            del sets
            torch.cuda.empty_cache()
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
