"""Matmul barrier kernel on the B200: bit-exactness against the reference's
sequential fp32 loop (sampled outputs) and throughput at BERT-base shapes.

    python tools/dot_check.py            # GPU box
Prints one JSON line per shape.
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_05213_b200 import host as H  # noqa: E402

SHAPES = [  # (name, batch dims, M, K, N, op)
    ("ffn_up", [], 32768, 768, 3072, "library_call"),
    ("qkv", [], 32768, 768, 768, "library_call"),
    ("scores", [768], 512, 64, 512, "batch_matmul"),
    ("ctx", [768], 512, 512, 64, "batch_matmul"),
    ("ragged", [3], 1000, 77, 333, "batch_matmul"),        # K % 4 != 0: the FMUL + FADD kernel
    ("ragged_packed", [3], 1000, 76, 332, "batch_matmul"),  # ragged tiles on the packed kernel
]


def seq_dot(a_row, b_col):
    acc = np.float32(0.0)
    for x, y in zip(a_row, b_col):
        acc = np.float32(acc + np.float32(np.float32(x) * np.float32(y)))
    return acc


def main():
    ctx = H.Context(0)
    for name, bd, M, K, N, op in SHAPES:
        ins = [{"id": "a", "op": "parameter", "shape": bd + [M, K]},
               {"id": "b", "op": "parameter", "shape": bd + [K, N]},
               {"id": "c", "op": op, "operands": ["a", "b"], "shape": bd + [M, N]}]
        if op == "library_call":
            ins[-1]["callee"] = "matmul"
        g = H.graph_from_json({"instructions": ins, "outputs": ["c"]})
        rep = H.CompileReport([], 0, 0, 1.0, ["c"])
        cg = H.CompiledGraph(ctx, g, rep)
        k = cg.barrier_kernels[0]
        a = torch.rand(bd + [M, K], device="cuda") * 2 - 1
        b = torch.rand(bd + [K, N], device="cuda") * 2 - 1
        c = torch.empty(bd + [M, N], device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            cg.run([a.data_ptr(), b.data_ptr()], [c.data_ptr()], stream=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            cg.run([a.data_ptr(), b.data_ptr()], [c.data_ptr()], stream=s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        batch = int(np.prod(bd)) if bd else 1
        flops = 2.0 * batch * M * N * K
        # bit-exact check on sampled outputs against the sequential fp32 loop
        rng = np.random.default_rng(0)
        A = a.reshape(batch, M, K)
        B = b.reshape(batch, K, N)
        C = c.reshape(batch, M, N)
        exact = 0
        samples = 48
        for _ in range(samples):
            bi, mi, ni = int(rng.integers(batch)), int(rng.integers(M)), int(rng.integers(N))
            want = seq_dot(A[bi, mi].cpu().numpy(), B[bi, :, ni].cpu().numpy())
            got = C[bi, mi, ni].item()
            exact += int(np.float32(got).tobytes() == want.tobytes())
        print(json.dumps({"shape": name, "batch": batch, "M": M, "K": K, "N": N, "ms": round(ms, 4),
                          "tflops": round(flops / ms / 1e9, 2), "bit_exact_samples": f"{exact}/{samples}",
                          "registers": k.info["registers"], "grid": k.info["grid"],
                          "packed": k.info["smem_bytes"] > 48 * 1024}), flush=True)
        cg.close()
        del a, b, c
    ctx.close()


if __name__ == "__main__":
    main()
