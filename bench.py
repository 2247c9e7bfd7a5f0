"""Benchmark: fused-graph effective HBM GB/s (% of peak) and kernel launches per graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
                    [--shard strong|weak]

One step = one execution of the whole compiled graph (every fusion group of
the reference plan = one stitched sm_100a launch) over one instance of the
named config with inputs resident in HBM.  Default workload: C5, the
BERT-base encoder-layer non-MatMul graph at batch 64, seq 512 (5 groups, 5.03
GB of compulsory traffic).

Multi-GPU, one process per GPU: `--shard strong` (default)
batch-shards ONE global instance — rank r of n runs the reference's plan of
its shard graph (workloads/plans/<C>.shard<n>.json, b64/n for C5; membership
equal to the global plan's, tests/test_shards.py) on its rows; the only
exchange is C3's batch-crossing column sum, combined across ranks inside the
column kernel over peer memory.  `--shard weak` runs a full replica per rank.
`value` = compulsory bytes of all ranks / max-over-ranks device time.
`--gpus N` without torchrun re-launches itself under torch.distributed.run.

`--impl reference` times the reference's own CPU executor (run_compiled,
built from the reference sources into oracle/_ref by oracle/Makefile; else
the C oracle port) on a bounded sample of the same workload whose reference
plan has the global plan's group membership (asserted), on all host cores
and on one core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Fused-graph effective HBM GB/s (% of peak) and kernel launches per graph"
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
WORKLOAD_NAMES = {
    "C1": "LayerNorm fp32 [8192,1024]",
    "C2": "Softmax fp32 [16,16,512,512]",
    "C3": "bias-add grad fp32 [65536,1024] (column reduce)",
    "C3b": "bias-add grad + dx output fp32 [65536,1024]",
    "C4": "transpose+bias+scale fp32 B32 S512 H16 D64",
    "C4b": "transpose+scale+bias fp32 B32 S512 H16 D64 (full bias)",
    "C4t": "key transpose [B,S,H,D]->[B,H,D,S]+bias+scale fp32 B32 S512 H16 D64 (extra, innermost-moving)",
    "C5": "BERT-base encoder-layer non-MatMul graph, batch 64 seq 512",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling (B200_PROFILING.md clocks line) read live by a thread,
    so the timed region can be bracketed by samples taken under the same load."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.rows = []  # (t, sm_mhz, max_mhz, reasons set)
        self.lock = threading.Lock()

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except Exception:
            self.proc = None
            return self
        threading.Thread(target=self._reader, daemon=True).start()
        return self

    def _reader(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                sm, mx = float(f[0]), float(f[1])
            except Exception:
                continue
            reasons = {n for n, v in zip(self.NAMES, f[4:8]) if v.lower().startswith("active")}
            with self.lock:
                self.rows.append((time.perf_counter(), sm, mx, reasons))

    def count_after(self, t):
        with self.lock:
            return sum(1 for r in self.rows if r[0] >= t)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t_lo, t_hi):
        with self.lock:
            rows = [r for r in self.rows if t_lo <= r[0] <= t_hi]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(r[1] for r in rows)
        reasons = set().union(*[r[3] for r in rows])
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": rows[0][2], "reasons": sorted(reasons),
                "samples": len(rows), "window_s": round(t_hi - t_lo, 3)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def plan_path(config, n=1, shard="strong"):
    """The plan a rank runs: the global plan, or (strong sharding over n > 1
    ranks) the reference's plan of one rank's shard graph."""
    if n == 1 or shard == "weak":
        return os.path.join(ROOT, "workloads", "plans", f"{config}.full.json")
    p = os.path.join(ROOT, "workloads", "plans", f"{config}.shard{n}.json")
    if not os.path.exists(p):
        raise SystemExit(f"bench.py: no {n}-way shard plan for {config} ({p}); shard counts: 2, 4, 8")
    return p


def membership(bundle):
    """Group membership of a plan bundle (what plan parity compares)."""
    return [(k["fusion_root"], sorted(k["members"]), list(k["roots"])) for k in bundle["kernels"]]


# --------------------------------------------------------------------------- reference arm

REF_FOOTPRINT = 64 << 20  # PipelineOptions::footprint_limit default (options.hpp)
_sample_cache = {}


def reference_sample(config):
    """A bounded sample of the same workload for the reference's CPU executor:
    the same rows (same lengths and op mix), fewer of them, planned by the
    reference with its footprint cap scaled to the sample (returns doc,
    description, footprint_limit).  The cap matters for C5 only: the reference
    merges the two LayerNorm groups when a whole group fits under it
    (fusion.cpp:69-85), so an unscaled sample would run a 4-group plan; the b8
    shard (4096 tokens) is the largest batch shard planned like b64 under the
    default 64 MiB, and the 64-token sample gets 64 MiB x 64/4096 = 1 MiB.
    reference_sample_plan() asserts the membership equals the global plan's."""
    from workloads import configs
    if config == "C5" and os.environ.get("SFX_REF_SAMPLE") == "b8":
        # the exact b8 shard (rank r's graph at 8 GPUs), default options: ~4 min
        # of single-core work per instance, for a one-off record
        return configs.c5_bert(B=8, S=512), "C5 b8 shard (1/8 of b64 s512, default options)", REF_FOOTPRINT
    if config == "C5":
        fl = REF_FOOTPRINT * 64 // 4096
        return (configs.c5_bert(B=1, S=512, Sq=64), "C5 query block: batch 1, 64 query rows x 512 keys "
                "(1/512 of b64 s512; footprint_limit 1 MiB = the b8 shard's 64 MiB scaled by 64/4096 tokens)", fl)
    sizes = {"C1": dict(R=64, C=1024), "C2": dict(B=1, H=1, S=128, L=512), "C3": dict(N=512, C=1024),
             "C3b": dict(N=512, C=1024), "C4": dict(B=1, S=128, H=16, D=64), "C4b": dict(B=1, S=128, H=16, D=64),
             "C4t": dict(B=1, S=128, H=16, D=64)}
    return configs.build(config, **sizes[config]), f"{config} at {sizes[config]}", REF_FOOTPRINT


def reference_sample_plan(config, path):
    """The reference's plan of the sample (ref_tool plan, same footprint cap the
    timing uses), checked against the global plan: same groups, same members."""
    if config in _sample_cache:
        return _sample_cache[config]
    doc, sample, fl = reference_sample(config)
    r = subprocess.run([REF_TOOL, "plan", path, "--footprint-limit", str(fl)], capture_output=True, text=True,
                       check=True)
    got = membership(json.loads(r.stdout))
    with open(plan_path(config)) as f:
        want = membership(json.load(f))
    if got != want:
        raise RuntimeError(f"reference plan of the {config} sample differs from the global plan: "
                           f"{[g[0] for g in got]} vs {[w[0] for w in want]}")
    _sample_cache[config] = len(got)
    return len(got)


def graph_bytes(doc):
    """Compulsory bytes: non-splat external inputs of each group once + roots once."""
    from paper_1811_05213_b200 import host as H
    g = H.parse_graph(doc)
    # parameters + outputs is exact for graphs whose groups are independent (all configs)
    b = sum(p.numel() * 4 for p in g.parameters())
    b += sum(g.at(o).numel() * 4 for o in g.outputs)
    return b


def time_reference_cpu(config, threads, iters=1):
    """One sample: `threads` independent run_compiled instances on as many host
    threads (the reference executor is single-threaded and reentrant)."""
    doc, sample, fl = reference_sample(config)
    nbytes = graph_bytes(doc)
    groups = None
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(doc, f)
        path = f.name
    try:
        if os.path.exists(REF_TOOL):
            groups = reference_sample_plan(config, path)
            r = subprocess.run([REF_TOOL, "bench", path, "42", str(threads), str(iters), "--footprint-limit", str(fl)],
                               capture_output=True, text=True, check=True)
            info = json.loads(r.stdout)
            if len(info["groups"]) != groups:
                raise RuntimeError(f"reference ran {len(info['groups'])} groups, planned {groups}")
            secs = info["seconds"]
            kind = "reference"
            execu = "reference run_compiled (oracle/_ref, built from the reference sources)"
        else:  # the C oracle port (dense interpreter restatement), single thread
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import sfx_testlib as T
            from paper_1811_05213_b200 import host as H
            g = H.parse_graph(doc)
            inputs = T.gen_inputs_fast(g, 42, -1.0, 1.0)
            t0 = time.perf_counter()
            for _ in range(iters):
                T.interpret(g, inputs, 0)
            secs = time.perf_counter() - t0
            threads = 1
            kind = "port"
            execu = "C oracle port of the reference interpreter"
    finally:
        os.unlink(path)
    gbs = threads * iters * nbytes / secs / 1e9
    cb = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": kind, "plan_groups": groups,
          "sample": f"{sample}; {execu}; {threads} independent instance(s) x {iters} iteration(s); "
                    f"{nbytes} compulsory bytes per instance; {secs:.2f} s wall"}
    return cb, secs


def cpu_baseline_both(config):
    """All host cores (throughput) and one core (the reference's own,
    single-threaded executor), on the same sample."""
    threads = os.cpu_count() or 1
    cb, secs = time_reference_cpu(config, threads)
    one, secs1 = time_reference_cpu(config, 1) if threads > 1 else (cb, secs)
    cb["value_1core"] = one["value"]
    cb["sample_1core"] = one["sample"]
    return cb, secs


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # W untimed samples, then K timed samples (each: one bounded sample of the
    # workload as independent instances on every host thread).  The whole run
    # is bounded to a few minutes: warm-ups stop after ~30 s, and the timed
    # samples are cut to what fits in ~150 s (reported as steps_timed).
    t0 = time.perf_counter()
    w_done = 0
    t_step = None
    while w_done < args.warmup and (w_done == 0 or time.perf_counter() - t0 < 30.0):
        _, t_step = time_reference_cpu(args.config, threads)
        w_done += 1
    k_run = max(1, min(args.steps, int(150.0 // max(t_step, 1e-3))))
    times, values, cb = [], [], None
    for _ in range(k_run):
        cb, secs = time_reference_cpu(args.config, threads)
        times.append(secs)
        values.append(cb["value"])
    ms = 1000.0 * sum(times) / len(times)
    # throughput over the timed samples: total bytes / total time
    value = sum(v * t for v, t in zip(values, times)) / sum(times)
    one, _ = time_reference_cpu(args.config, 1) if threads > 1 else (cb, None)
    cb = dict(cb, value=value, value_1core=one["value"], sample_1core=one["sample"])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "steps_timed": k_run, "warmup_run": w_done,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling_of(args), "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_obj(args.config, args.gpus, args.combine, args.shard),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": (f"CPU reference: each step is one bounded sample on {threads} host threads; "
                 f"{k_run} of the {args.steps} requested steps timed, {w_done} warm-up(s), to keep the run "
                 "within a few minutes"),
    }
    print(json.dumps(line), flush=True)
    return 0


def agreed_rounds(more, round_fn, ws, red_dev):
    """Run round_fn while more() holds on ANY rank: every rank runs the same
    number of rounds, so a step that exchanges data across ranks (the
    cross-rank column combine) is issued equally often everywhere."""
    import torch
    import torch.distributed as dist
    n = 0
    while True:
        m = bool(more())
        if ws > 1:
            flag = torch.tensor([1.0 if m else 0.0], device=red_dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            m = flag.item() > 0
        if not m:
            return n
        round_fn()
        n += 1


def scaling_of(args):
    return "strong" if args.shard == "strong" else "weak"


def config_obj(config, n, combine="peer", shard="strong"):
    """The workload (identical on both arms); run details go in `run`."""
    from workloads import configs
    strong = shard == "strong" and n > 1
    if strong:
        per = configs.shard_sizes(config, n)
        d = configs.SHARD_DIM[config]
        par = f"one global instance batch-sharded over {n} GPUs along {d} ({d}={per[d]} per rank)"
    else:
        par = f"independent graph instances x{n} (one full instance per GPU)" if n > 1 else "1 GPU"
    if config in ("C3", "C3b") and n > 1:
        par += ("; column sums combined across ranks inside the column kernel (peer memory)" if combine == "peer"
                else "; NCCL all-reduce of the column sums")
    else:
        par += "; no collective"
    c = {"workload": f"{config}: {WORKLOAD_NAMES[config]}",
         "plan": os.path.relpath(plan_path(config, n, shard), ROOT) + " (reference compile_graph, default "
                 "PipelineOptions)",
         "parallelism": par}
    if strong:
        c["shard"] = {"dim": configs.SHARD_DIM[config], "ranks": n, "per_rank": configs.shard_sizes(config, n),
                      "global": configs.FULL[config]}
    return c


# --------------------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1811_05213_b200 import host as H

    ws, rank, local = dist_env()
    # one process per GPU; the modulo only matters for smoke-testing the
    # multi-rank path with more ranks than GPUs (--dist-backend gloo)
    local = local % max(1, torch.cuda.device_count())
    if ws > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if args.dist_backend == "nccl" else "cpu"  # where cross-rank reductions of scalars live
    ctx = H.Context(local)
    g, rep, bundle = H.load_bundle(plan_path(args.config, ws, args.shard))
    # the one batch-crossing exchange on this path is a column reduction over
    # the batch (C3's db).  Default: the column kernel combines the ranks'
    # partials itself through peer memory (cross_rank); --combine nccl runs
    # the unfused baseline (kernel, then ncclAllReduce of the column sums).
    # (only graphs with a reduction over the batch dim need the peer group)
    batch_reduce = any(i.op == "reduce" and 0 in i.reduce_dims for i in g.instructions)
    peer = ws > 1 and args.combine == "peer" and batch_reduce
    if peer:
        ctx.peer_init(rank, ws, H.torch_all_gather)
    cg = H.CompiledGraph(ctx, g, rep, cross_rank=int(peer))
    kinfo = [k.info for k in cg.kernels]
    n_kernels = len(cg.kernels)

    # inputs resident in HBM; enough rotating sets that the sets exceed L2 (126 MB)
    per_set = sum(g.at(p).numel() * 4 for p in cg.param_ids) + sum(g.at(o).numel() * 4 for o in g.outputs)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    # (small per-rank shards at 8 GPUs need many sets: C1 at 8 ranks is 8.4 MB)
    nsets = max(1, min(64, math.ceil(3 * l2 / per_set)))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    sets = []
    for _ in range(nsets):
        ins = [torch.rand(g.at(p).shape, generator=gen, device=dev, dtype=torch.float32) * 2 - 1
               for p in cg.param_ids]
        outs = [torch.empty(g.at(o).shape, device=dev, dtype=torch.float32) for o in g.outputs]
        sets.append(([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], ins, outs))
    stream = torch.cuda.Stream(device=dev)
    algo_bytes = sum(k["algorithmic_bytes"] for k in kinfo)

    # the one batch-crossing exchange on this path: column sums (C3's db) of
    # every rank's batch shard are combined with an NCCL all-reduce of C floats
    colsum_outputs = []
    if ws > 1 and not peer:
        for k in cg.kernels:
            if k.info["strategy"] == "col":
                for r in k.program.roots:
                    if r in g.outputs and g.at(r).numel() < sum(g.at(x).numel() for x in k.input_ids):
                        colsum_outputs.append(g.outputs.index(r))
    if colsum_outputs:
        uid = [H.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], ws, rank)

    # independent graph instances in flight on separate streams (SURVEY §7
    # hard part 5): small graphs otherwise expose launch/ramp/tail latency.
    # Concurrent instances always use distinct buffer sets; kernels that own a
    # workspace (cross-CTA column combine) run one instance at a time.
    # Two instances for graphs above 512 MB (C5 and its shards: the next
    # instance's first kernels run under the previous one's last ramp-down;
    # measured C5 b8 shard 0.097 -> 0.091 ms per graph), four below.  Kernels
    # with a cross-CTA workspace (column combine) get one workspace per stream
    # and per captured graph, so they run concurrently too; kernels that
    # exchange with peer ranks run one instance at a time (every rank must
    # issue them in the same order).
    has_peer = peer
    inflight = args.inflight if args.inflight > 0 else (4 if per_set <= (512 << 20) else 2 if per_set <= (16 << 30) else 1)
    if has_peer:
        inflight = 1
    inflight = max(1, inflight)
    while len(sets) < inflight:  # never share a buffer set between concurrent instances
        ins = [torch.rand(g.at(p).shape, generator=gen, device=dev, dtype=torch.float32) * 2 - 1
               for p in cg.param_ids]
        outs = [torch.empty(g.at(o).shape, device=dev, dtype=torch.float32) for o in g.outputs]
        sets.append(([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], ins, outs))
    nsets = len(sets)
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(inflight - 1)]
    torch.cuda.synchronize(dev)  # inputs were written on torch's stream; ours do not wait for it

    def step(i):
        s = streams[i % inflight]
        pi, po, _, outs = sets[i % nsets]
        cg.run(pi, po, stream=s.cuda_stream, cuda_graph=True)
        for oi in colsum_outputs:
            ctx.allreduce_sum_f32(po[oi], outs[oi].numel(), s.cuda_stream)

    def fork():
        ev = torch.cuda.Event()
        ev.record(stream)
        for s in streams[1:]:
            s.wait_event(ev)

    def join():
        for s in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            stream.wait_event(ev)

    clk = Clocks(local).start()
    fork()
    for i in range(args.warmup):
        step(i)
    join()
    torch.cuda.synchronize(dev)
    # keep the GPU under the same load until the sampler is producing samples,
    # so the timed region is bracketed by clock samples taken under load
    # Ranks run the same number of load rounds: a step that exchanges data
    # across ranks (the cross-rank column combine) must be issued equally often
    # on every rank, so the continue decision is agreed each round (max).
    t_load = time.perf_counter()
    n_load = 0
    def load_round():
        nonlocal n_load
        for _ in range(16):
            step(n_load)
            n_load += 1
        torch.cuda.synchronize(dev)
    agreed_rounds(lambda: clk.count_after(t_load + 0.15) < 2 and time.perf_counter() - t_load < 5.0,
                  load_round, ws, red_dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count()
    t_lo = time.perf_counter()
    e0.record(stream)
    fork()
    for i in range(args.steps):
        step(i)
    join()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t_hi = time.perf_counter()
    launches = ctx.launch_count() - launches0
    t_post = time.perf_counter()
    agreed_rounds(lambda: clk.count_after(t_post) < 2 and time.perf_counter() - t_post < 3.0,
                  load_round, ws, red_dev)
    clk.stop()
    # samples within 150 ms of the timed region, all under continuous load of the same step
    clocks = clk.summary(t_lo - 0.15, max(t_hi, t_post) + 0.15)
    clocks["note"] = "sampled every 50 ms under continuous load of this step bracketing the timed region"
    if ws > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=red_dev)
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # per-kernel live timing on the launching stream (roofline of each group)
    per_kernel = []
    scratch = {}
    reps = max(3, min(20, args.steps))
    for ki, k in enumerate(cg.kernels):
        slots = {pid: i for i, pid in enumerate(cg.param_ids)}
        outs_slot = {o: i for i, o in enumerate(g.outputs)}
        # tensors between groups (neither params nor graph outputs) get scratch buffers
        for x in list(k.input_ids) + list(k.program.roots):
            if x not in slots and x not in outs_slot and x not in scratch:
                scratch[x] = torch.zeros(g.at(x).shape, device=dev, dtype=torch.float32)

        def ptrs(sidx):
            pi, po, _, _ = sets[sidx % nsets]
            pick_in = lambda x: pi[slots[x]] if x in slots else scratch[x].data_ptr()  # noqa: E731
            pick_out = lambda x: po[outs_slot[x]] if x in outs_slot else scratch[x].data_ptr()  # noqa: E731
            return [pick_in(x) for x in k.input_ids], [pick_out(r) for r in k.program.roots]

        for i in range(2):
            a, b = ptrs(i)
            k.launch(a, b, stream.cuda_stream)
        # (1) average launch duration as the kernel runs in the timed region:
        # `reps` back-to-back launches (rotating buffer sets, PDL-chained) between
        # two events; (2) for reference, each launch bracketed by its own events
        # (every launch then also pays the launch latency the chain hides)
        eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eb0.record(stream)
        for i in range(reps):
            a, b = ptrs(i)
            k.launch(a, b, stream.cuda_stream)
        eb1.record(stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i in range(reps):
            a, b = ptrs(i)
            ev[i][0].record(stream)
            k.launch(a, b, stream.cuda_stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        avg = eb0.elapsed_time(eb1) / reps
        avg_isolated = sum(s.elapsed_time(e) for s, e in ev) / reps
        # context: a device copy of the same byte count (half read, half
        # written) as one launch — the achievable single-launch time at this size
        half = k.info["algorithmic_bytes"] // 8
        cps = [(torch.empty(half, device=dev), torch.empty(half, device=dev)) for _ in range(2)]
        for i in range(2):
            with torch.cuda.stream(stream):
                cps[i % 2][1].copy_(cps[i % 2][0])
        cb0, cb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):  # back to back, like the kernel's launches above
            cb0.record(stream)
            for i in range(reps):
                cps[i % 2][1].copy_(cps[i % 2][0])
            cb1.record(stream)
        torch.cuda.synchronize(dev)
        copy_ms = cb0.elapsed_time(cb1) / reps
        del cps
        per_kernel.append({"group": k.program.fusion_root, "kernel": k.info["entry"],
                           "strategy": k.info["strategy"], "ms": avg, "ms_isolated_launch": avg_isolated,
                           "gbs_isolated_launch": k.info["algorithmic_bytes"] / (avg_isolated * 1e-3) / 1e9,
                           "bytes": k.info["algorithmic_bytes"],
                           "gbs": k.info["algorithmic_bytes"] / (avg * 1e-3) / 1e9,
                           "same_size_copy_ms": copy_ms, "vs_same_size_copy": copy_ms / avg,
                           "grid": k.info["grid"], "block": k.info["block"], "regs": k.info["registers"]})

    # end-to-end through the reference-facing host-buffer call (TensorValue in/out)
    pin_in = [torch.empty(g.at(p).shape, dtype=torch.float32).pin_memory() for p in cg.param_ids]
    for t, d in zip(pin_in, sets[0][2]):
        t.copy_(d.cpu())
    pin_out = {o: torch.empty(g.at(o).shape, dtype=torch.float32).pin_memory() for o in g.outputs}
    import ctypes as C
    pin_arr = (C.c_void_p * len(pin_in))(*[t.data_ptr() for t in pin_in])
    out_arr = (C.c_void_p * len(g.outputs))(*[pin_out[o].data_ptr() for o in g.outputs])
    h2d = sum(t.numel() * 4 for t in pin_in)
    d2h = sum(t.numel() * 4 for t in pin_out.values())

    # a second pinned output set: consecutive pipelined steps write different host buffers
    pin_out2 = {o: torch.empty(g.at(o).shape, dtype=torch.float32).pin_memory() for o in g.outputs}
    out_arr2 = (C.c_void_p * len(g.outputs))(*[pin_out2[o].data_ptr() for o in g.outputs])

    def e2e_step():
        H._check(H.lib().sfx_graph_run_host(cg.h, pin_arr, len(pin_in), out_arr, len(g.outputs),
                                             C.c_void_p(stream.cuda_stream)))

    def e2e_step_async(i):
        H._check(H.lib().sfx_graph_run_host_async(cg.h, pin_arr, len(pin_in), out_arr if i % 2 == 0 else out_arr2,
                                                   len(g.outputs), C.c_void_p(stream.cuda_stream)))

    def timed_max(fn, n):
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        fn(n)
        sec = (time.perf_counter() - t0) / n
        t = torch.tensor([sec], device=red_dev)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sync_run(n):
        for _ in range(n):
            e2e_step()

    def async_run(n):
        for i in range(n):
            e2e_step_async(i)
        stream.synchronize()

    e2e_step()
    async_run(2)
    e2e_steps = max(2, min(5, args.steps))
    e2e_sync_s = timed_max(sync_run, e2e_steps)
    # headline: consecutive steps pipelined through sfx_graph_run_host_async
    # (step i+1's host->device copies overlap step i's kernels and copies back);
    # every step still copies its inputs in and its outputs out
    e2e_s = timed_max(async_run, max(4, min(10, args.steps)))
    host_ok = all(torch.equal(pin_out[o], pin_out2[o]) for o in g.outputs)

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_kind = peaks()
    total_bytes = algo_bytes * ws
    value = total_bytes / (ms_max * 1e-3) / 1e9
    dom = max(per_kernel, key=lambda r: r["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}/{dom['kernel']}")
    except Exception:
        pass
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            cpu, _ = cpu_baseline_both(args.config)
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": scaling_of(args),
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.rand U(-1,1) inputs resident in HBM)",
        "config": config_obj(args.config, ws, args.combine, args.shard),
        "run": {"l2_policy": f"{nsets} rotating input/output set(s) of {per_set / 1e6:.1f} MB per rank "
                             f"({nsets * per_set / 1e6:.0f} MB > L2 {l2 / 1e6:.0f} MB)",
                "groups": n_kernels, "launches_per_graph": n_kernels, "instances_in_flight": inflight,
                "bytes_per_rank_per_step": algo_bytes, "ranks": ws},
        "pct_of_peak": 100.0 * value / ws / peak,
        "peak_gbs": peak, "peak_kind": peak_kind,
        "kernel_launches_per_graph": n_kernels,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                     "frac": dom["gbs"] / peak, "traffic": traffic, "kernel": dom["kernel"],
                     "algorithmic_bytes_per_launch": dom["bytes"], "ms_per_launch": dom["ms"],
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
        "per_kernel": per_kernel,
        "e2e": {"value": total_bytes / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                "path": "sfx_graph_run_host_async, consecutive steps pipelined (pinned host buffers; every step: "
                        "H2D of its inputs + 1 launch per group + D2H of its outputs)",
                "ms_per_step_synchronous": e2e_sync_s * 1e3,
                "value_synchronous": total_bytes / e2e_sync_s / 1e9,
                "alternating_output_sets_identical": host_ok},
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """`--gpus N` without torchrun: re-run this script as N ranks under
    torch.distributed.run (127.0.0.1 rendezvous) and relay rank 0's line."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOAD_NAMES))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for the barrier / max-over-ranks timing (nccl on GPUs)")
    ap.add_argument("--combine", default="peer", choices=["peer", "nccl"],
                    help="cross-rank column sums: fused into the column kernel over peer memory, or NCCL after it")
    ap.add_argument("--inflight", type=int, default=0,
                    help="independent graph instances in flight per GPU (0 = auto)")
    ap.add_argument("--shard", default="strong", choices=["strong", "weak"],
                    help="strong: one global instance batch-sharded over the ranks (SURVEY §8(e)); "
                         "weak: a full instance per rank")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
