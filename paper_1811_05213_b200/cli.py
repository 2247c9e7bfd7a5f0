"""`run --device`: the reference CLI's `run` subcommand on the B200 executor.

    python -m paper_1811_05213_b200.cli run <plan.json> --inputs <inputs.json> [--dump-values] [--strategy auto]
    python -m paper_1811_05213_b200.cli plan-info <plan.json>

Mirrors `stitchfuse run G --inputs I` (reference tools/stitchfuse.cpp:231-249):
the same inputs file format (`load_inputs`, stitchfuse.cpp:52-88: an object of
id -> {shape, dtype, data | random_seed}; random tensors drawn exactly like the
reference, std::mt19937_64 + uniform_real_distribution<float>(-1,1) /
uniform_int_distribution<int32_t>(-4,4) as implemented by libstdc++ 13), the same
output lines (`<id> shape=[..]f32 checksum=<sum>`, value_checksum
stitchfuse.cpp:90-98) and exit codes (0 ok, 1 user error, 2 internal error,
stitchfuse.cpp:290-303).  The plan is the reference's own: a plan bundle from
`compile_graph` (e.g. `oracle/_ref/ref_tool plan G`, or workloads/plans/*.json);
this tool never re-plans.  Every fused group runs as one sm_100a launch.
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import host as H

M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++11 standard parameters), vectorised twist."""

    N, M = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UPPER, LOWER = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [0] * self.N
        mt[0] = seed & M64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & M64
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        with np.errstate(over="ignore"):
            def step(lo, hi):
                y = (mt[lo:hi] & self.UPPER) | (mt[lo + 1:hi + 1] & self.LOWER)
                return (y >> np.uint64(1)) ^ np.where((y & np.uint64(1)) != 0, self.MATRIX_A, np.uint64(0))
            mt[0:N - M] = mt[M:N] ^ step(0, N - M)
            mt[N - M:N - 1] = mt[0:M - 1] ^ step(N - M, N - 1)
            y = (mt[N - 1] & self.UPPER) | (mt[0] & self.LOWER)
            mt[N - 1] = mt[M - 1] ^ (y >> np.uint64(1)) ^ (self.MATRIX_A if int(y) & 1 else np.uint64(0))
        self.idx = 0

    def take(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self.idx >= self.N:
                self._twist()
            c = min(n - k, self.N - self.idx)
            out[k:k + c] = self.mt[self.idx:self.idx + c]
            self.idx += c
            k += c
        x = out
        x = x ^ ((x >> np.uint64(29)) & np.uint64(0x5555555555555555))
        x = x ^ ((x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        x = x ^ ((x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        x = x ^ (x >> np.uint64(43))
        return x

    def next(self) -> int:
        return int(self.take(1)[0])


def uniform_float(rng: MT19937_64, n: int, a: float, b: float) -> np.ndarray:
    """uniform_real_distribution<float>(a, b): generate_canonical<float, 24>
    (random.tcc:3349-3381) then `canon * (b - a) + a` in float."""
    x = rng.take(n)
    ret = x.astype(np.float32) / np.float32(2.0 ** 64)
    ret = np.where(ret >= np.float32(1), np.nextafter(np.float32(1), np.float32(0)), ret).astype(np.float32)
    return (ret * np.float32(np.float32(b) - np.float32(a)) + np.float32(a)).astype(np.float32)


def uniform_int(rng: MT19937_64, n: int, a: int, b: int) -> np.ndarray:
    """uniform_int_distribution<int32_t>(a, b) with a 64-bit engine: Lemire's
    nearly-divisionless downscaling in 128-bit (uniform_int_dist.h:257-281)."""
    rng_range = (b - a + 1)
    threshold = ((1 << 64) - rng_range) % rng_range
    out = np.empty(n, dtype=np.int32)
    for i in range(n):
        prod = rng.next() * rng_range
        while (prod & M64) < rng_range and (prod & M64) < threshold:
            prod = rng.next() * rng_range
        out[i] = (prod >> 64) + a
    return out


class UserError(Exception):
    pass


def load_inputs(path: str, graph: H.TensorGraph, base_seed: int = 0) -> dict:
    """stitchfuse.cpp:52-88."""
    try:
        doc = json.load(open(path))
    except (OSError, ValueError) as e:
        raise UserError(f"{path}: {e}")
    out = {}
    for key, j in doc.items():
        shape = list(j["shape"])
        dtype = j.get("dtype", "f32")
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        if "data" in j:
            data = j["data"]
            if len(data) != n:
                raise UserError(f"{path}: {key}: data size mismatch")
            arr = np.array(data, dtype=np.float64)
            arr = arr.astype(np.float32) if dtype != "i32" else arr.astype(np.int64).astype(np.int32)
        else:
            rng = MT19937_64(int(j.get("random_seed", base_seed)))
            arr = uniform_float(rng, n, -1.0, 1.0) if dtype != "i32" else uniform_int(rng, n, -4, 4)
        if key not in graph.index:
            raise UserError(f"{path}: unknown input id {key}")
        out[key] = arr.reshape(shape)
    return out


def value_checksum(a: np.ndarray) -> float:
    """stitchfuse.cpp:90-98: sequential double sum."""
    s = 0.0
    for v in np.asarray(a, dtype=np.float64).ravel():
        s += float(v)
    return s


def fmt_shape(ins) -> str:
    return "[" + ",".join(str(d) for d in ins.shape) + "]" + ins.dtype


def fmt_num(x: float) -> str:
    return f"{x:.6g}"


def cmd_run(args) -> int:
    graph, report, bundle = H.load_bundle(args.plan)
    inputs = load_inputs(args.inputs, graph, args.seed)
    for p in graph.parameters():
        if p.id not in inputs:
            raise H.ExecError("missing input for parameter " + p.id)
    values = H.run_compiled(report, graph, inputs, strategy=args.strategy)
    for o in graph.outputs:
        v = values[o]
        print(f"{o} shape={fmt_shape(graph.at(o))} checksum={fmt_num(value_checksum(v))}")
        if args.dump_values:
            vals = v.ravel()
            print("  " + " ".join((f"{x:.6f}" if v.dtype == np.float32 else str(int(x))) for x in vals))
    return 0


def cmd_plan_info(args) -> int:
    graph, report, bundle = H.load_bundle(args.plan)
    print(f"baseline_kernels: {bundle['baseline_kernels']}")
    print(f"fused_kernels: {bundle['fused_kernels']}")
    print(f"fusion_ratio: {bundle['fusion_ratio']:.6g}")
    for k in report.kernels:
        src, cubin, note = H.codegen(graph, k.program, args.strategy)
        print(f"computation {k.program.fusion_root}: members={len(k.program.members)} roots={','.join(k.program.roots)}"
              f" -> {note}")
    for u in bundle.get("unfused", []):
        print(f"standalone {u} ({graph.at(u).op})")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="stitchfuse-device")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="execute a planned graph on the B200")
    r.add_argument("plan", help="plan bundle (reference compile_graph output)")
    r.add_argument("--inputs", required=True)
    r.add_argument("--dump-values", action="store_true")
    r.add_argument("--seed", type=int, default=0, help="default random_seed (reference --seed)")
    r.add_argument("--strategy", default="auto", choices=sorted(H.STRATEGIES))
    p = sub.add_parser("plan-info", help="per-group lowering of a plan bundle (no GPU needed)")
    p.add_argument("plan")
    p.add_argument("--strategy", default="auto", choices=sorted(H.STRATEGIES))
    args = ap.parse_args(argv)
    try:
        return cmd_run(args) if args.cmd == "run" else cmd_plan_info(args)
    except UserError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except H.ExecError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1 if e.status in (1,) else 2
    except Exception as e:  # noqa: BLE001
        print(f"internal error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
