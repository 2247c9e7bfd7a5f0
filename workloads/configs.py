"""The five BASELINE.json workloads as graphs in the reference's JSON graph format.

Graph format: the reference parser's key set (`ir.cpp:332-378`): `id`, `op`,
`operands`, `shape`, `dtype`, `permutation`, `reduce_dims`, `reducer`,
`broadcast_dim_map`, `scalar`, `value`, plus top-level `instructions` /
`outputs`.  `reducer: "mean"` is lowered by the reference parser to
`<id>.sum` + `scale(1/n)` (`ir.cpp:396-428`).  The graphs follow SURVEY.md
Appendix A exactly; the fusion plans executed for them are produced by the
reference's own `compile_graph` (`pipeline.cpp:18-63`) and committed next to
them by `workloads/make_workloads.py`.

C1 LayerNorm [R,C]; C2 softmax [B,H,S,S]; C3 bias-grad [N,C] (C3b adds the
dx output); C4 transpose+bias+scale [B,S,H,D] (C4b full-bias form); C5
BERT-base encoder-layer non-MatMul graph at batch B, seq S.
"""

from __future__ import annotations

import json


class _G:
    def __init__(self):
        self.instrs = []

    def add(self, id, op, operands=(), shape=(), **attrs):
        j = {"id": id, "op": op, "shape": list(shape)}
        if operands:
            j["operands"] = list(operands)
        j.update(attrs)
        self.instrs.append(j)
        return id

    def param(self, id, shape):
        return self.add(id, "parameter", (), shape)

    def doc(self, outputs):
        return {"instructions": self.instrs, "outputs": list(outputs)}


def _layernorm(g: _G, x, gamma, beta, R, C, prefix, out):
    p = prefix
    g.add(p + "mean", "reduce", [x], [R], reduce_dims=[1], reducer="mean")
    g.add(p + "mean_b", "broadcast", [p + "mean"], [R, C], broadcast_dim_map=[0])
    g.add(p + "d", "sub", [x, p + "mean_b"], [R, C])
    g.add(p + "d2", "mul", [p + "d", p + "d"], [R, C])
    g.add(p + "var", "reduce", [p + "d2"], [R], reduce_dims=[1], reducer="mean")
    g.add(p + "eps", "constant", [], [R], value=1e-5)
    g.add(p + "ve", "add", [p + "var", p + "eps"], [R])
    g.add(p + "rstd", "rsqrt", [p + "ve"], [R])
    g.add(p + "rstd_b", "broadcast", [p + "rstd"], [R, C], broadcast_dim_map=[0])
    g.add(p + "n", "mul", [p + "d", p + "rstd_b"], [R, C])
    g.add(p + "gamma_b", "broadcast", [gamma], [R, C], broadcast_dim_map=[1])
    g.add(p + "beta_b", "broadcast", [beta], [R, C], broadcast_dim_map=[1])
    g.add(p + "ng", "mul", [p + "n", p + "gamma_b"], [R, C])
    g.add(out, "add", [p + "ng", p + "beta_b"], [R, C])


def _softmax(g: _G, s, shape, prefix, out):
    p = prefix
    rows = list(shape[:-1])
    keep = list(range(len(rows)))
    last = len(shape) - 1
    g.add(p + "max", "reduce", [s], rows, reduce_dims=[last], reducer="max")
    g.add(p + "max_b", "broadcast", [p + "max"], shape, broadcast_dim_map=keep)
    g.add(p + "z", "sub", [s, p + "max_b"], shape)
    g.add(p + "e", "exp", [p + "z"], shape)
    g.add(p + "sum", "reduce", [p + "e"], rows, reduce_dims=[last], reducer="sum")
    g.add(p + "sum_b", "broadcast", [p + "sum"], shape, broadcast_dim_map=keep)
    g.add(out, "div", [p + "e", p + "sum_b"], shape)


def c1_layernorm(R=8192, C=1024):
    g = _G()
    g.param("x", [R, C])
    g.param("gamma", [C])
    g.param("beta", [C])
    _layernorm(g, "x", "gamma", "beta", R, C, "ln.", "y")
    return g.doc(["y"])


def c2_softmax(B=16, H=16, S=512, L=512):
    g = _G()
    shape = [B, H, S, L]
    g.param("s", shape)
    _softmax(g, "s", shape, "sm.", "y")
    return g.doc(["y"])


def c3_biasgrad(N=65536, C=1024, with_dx=False):
    g = _G()
    g.param("dy", [N, C])
    g.param("x", [N, C])
    g.add("zero", "constant", [], [N, C], value=0.0)
    g.add("mask", "compare", ["x", "zero"], [N, C])
    g.add("dx", "mul", ["dy", "mask"], [N, C])
    g.add("db", "reduce", ["dx"], [C], reduce_dims=[0], reducer="sum")
    outs = ["db"]
    if with_dx:
        g.add("dx_out", "scale", ["dx"], [N, C], scalar=1.0)
        outs.append("dx_out")
    return g.doc(outs)


def c4_transpose(B=32, S=512, H=16, D=64):
    g = _G()
    g.param("x", [B, S, H, D])
    g.param("bias", [H, D])
    g.add("bias_b", "broadcast", ["bias"], [B, S, H, D], broadcast_dim_map=[2, 3])
    g.add("xb", "add", ["x", "bias_b"], [B, S, H, D])
    g.add("xt", "transpose", ["xb"], [B, H, S, D], permutation=[0, 2, 1, 3])
    g.add("y", "scale", ["xt"], [B, H, S, D], scalar=0.125)
    return g.doc(["y"])


def c4t_transpose(B=32, S=512, H=16, D=64):
    """Extra (not a BASELINE.json config): the attention key transpose
    [B,S,H,D] -> [B,H,D,S], which moves the innermost dimension — exercises the
    shared-memory-tiled transpose template at the C4 size."""
    g = _G()
    g.param("x", [B, S, H, D])
    g.param("bias", [H, D])
    g.add("bias_b", "broadcast", ["bias"], [B, S, H, D], broadcast_dim_map=[2, 3])
    g.add("xb", "add", ["x", "bias_b"], [B, S, H, D])
    g.add("xt", "transpose", ["xb"], [B, H, D, S], permutation=[0, 2, 3, 1])
    g.add("y", "scale", ["xt"], [B, H, D, S], scalar=0.125)
    return g.doc(["y"])


def c4b_transpose(B=32, S=512, H=16, D=64):
    g = _G()
    g.param("q", [B, S, H, D])
    g.param("bias", [B, H, S, D])
    g.add("qt", "transpose", ["q"], [B, H, S, D], permutation=[0, 2, 1, 3])
    g.add("qs", "scale", ["qt"], [B, H, S, D], scalar=0.125)
    g.add("y", "add", ["qs", "bias"], [B, H, S, D])
    return g.doc(["y"])


def c5_bert(B=64, S=512, Hd=768, NH=12, FF=3072, Sq=None):
    """Sq < S builds a query block of the same layer (rows of identical length
    and type, byte mix identical to the full layer) — the bounded CPU sample."""
    Sq = S if Sq is None else Sq
    D = Hd // NH
    T = B * Sq
    g = _G()
    att = [B, NH, Sq, S]
    # attention scores -> scaled, masked softmax -> dropout mask
    g.param("scores", att)
    g.param("amask", att)
    g.param("dmask_a", att)
    g.add("scores_s", "scale", ["scores"], att, scalar=0.125)
    g.add("scores_m", "add", ["scores_s", "amask"], att)
    _softmax(g, "scores_m", att, "sm.", "probs")
    g.add("probs_d", "mul", ["probs", "dmask_a"], att)
    # context head merge
    g.param("ctx", [B, NH, Sq, D])
    g.add("ctx_t", "transpose", ["ctx"], [B, Sq, NH, D], permutation=[0, 2, 1, 3])
    g.add("ctx_r", "reshape", ["ctx_t"], [T, Hd])
    # attention output bias + dropout + residual + LayerNorm 1
    for p in ("attn_o", "dmask_o", "resid_in"):
        g.param(p, [T, Hd])
    for p in ("b_o", "g1", "be1"):
        g.param(p, [Hd])
    g.add("b_o_b", "broadcast", ["b_o"], [T, Hd], broadcast_dim_map=[1])
    g.add("attn_ob", "add", ["attn_o", "b_o_b"], [T, Hd])
    g.add("attn_od", "mul", ["attn_ob", "dmask_o"], [T, Hd])
    g.add("res1", "add", ["attn_od", "resid_in"], [T, Hd])
    _layernorm(g, "res1", "g1", "be1", T, Hd, "ln1.", "h1")
    # FFN1 bias + tanh-GELU
    g.param("ff1", [T, FF])
    g.param("b_f1", [FF])
    g.add("b_f1_b", "broadcast", ["b_f1"], [T, FF], broadcast_dim_map=[1])
    g.add("u", "add", ["ff1", "b_f1_b"], [T, FF])
    g.add("u2", "mul", ["u", "u"], [T, FF])
    g.add("u3", "mul", ["u2", "u"], [T, FF])
    g.add("u3s", "scale", ["u3"], [T, FF], scalar=0.044715)
    g.add("inner", "add", ["u", "u3s"], [T, FF])
    g.add("inner_s", "scale", ["inner"], [T, FF], scalar=0.7978845608028654)
    g.add("th", "tanh", ["inner_s"], [T, FF])
    g.add("one", "constant", [], [T, FF], value=1.0)
    g.add("th1", "add", ["th", "one"], [T, FF])
    g.add("half_u", "scale", ["u"], [T, FF], scalar=0.5)
    g.add("gelu", "mul", ["half_u", "th1"], [T, FF])
    # FFN2 bias + dropout + residual + LayerNorm 2
    for p in ("ff2", "dmask_f", "h1_in"):
        g.param(p, [T, Hd])
    for p in ("b_f2", "g2", "be2"):
        g.param(p, [Hd])
    g.add("b_f2_b", "broadcast", ["b_f2"], [T, Hd], broadcast_dim_map=[1])
    g.add("ff2b", "add", ["ff2", "b_f2_b"], [T, Hd])
    g.add("ff2d", "mul", ["ff2b", "dmask_f"], [T, Hd])
    g.add("res2", "add", ["ff2d", "h1_in"], [T, Hd])
    _layernorm(g, "res2", "g2", "be2", T, Hd, "ln2.", "h2")
    return g.doc(["probs_d", "ctx_r", "h1", "gelu", "h2"])


def c5_layer(B=64, S=512, Hd=768, NH=12, FF=3072):
    """Extra (not a BASELINE.json config): the whole BERT-base encoder layer
    with its matmuls as instructions — LibraryCall "matmul" for the dense
    projections, BatchMatMul for the attention products — so the reference
    planner chains the C5 groups through matmul barriers.
    The non-matmul part is C5's graph; inputs are the hidden states x and the
    weights, plus C5's attention mask and dropout masks."""
    D = Hd // NH
    T = B * S
    att = [B, NH, S, S]
    g = _G()
    g.param("x", [T, Hd])
    for w in ("q", "k", "v"):
        g.param("W" + w, [Hd, Hd])
        g.param("b" + w, [Hd])
        g.add(w + "_mm", "library_call", ["x", "W" + w], [T, Hd], callee="matmul")
        g.add("b%s_b" % w, "broadcast", ["b" + w], [T, Hd], broadcast_dim_map=[1])
        g.add(w + "_b", "add", [w + "_mm", "b%s_b" % w], [T, Hd])
        g.add(w + "_r", "reshape", [w + "_b"], [B, S, NH, D])
    g.add("q_t", "transpose", ["q_r"], [B, NH, S, D], permutation=[0, 2, 1, 3])
    g.add("k_t", "transpose", ["k_r"], [B, NH, D, S], permutation=[0, 2, 3, 1])
    g.add("v_t", "transpose", ["v_r"], [B, NH, S, D], permutation=[0, 2, 1, 3])
    g.add("scores", "batch_matmul", ["q_t", "k_t"], att)
    g.param("amask", att)
    g.param("dmask_a", att)
    g.add("scores_s", "scale", ["scores"], att, scalar=0.125)
    g.add("scores_m", "add", ["scores_s", "amask"], att)
    _softmax(g, "scores_m", att, "sm.", "probs")
    g.add("probs_d", "mul", ["probs", "dmask_a"], att)
    g.add("ctx", "batch_matmul", ["probs_d", "v_t"], [B, NH, S, D])
    g.add("ctx_t", "transpose", ["ctx"], [B, S, NH, D], permutation=[0, 2, 1, 3])
    g.add("ctx_r", "reshape", ["ctx_t"], [T, Hd])
    g.param("Wo", [Hd, Hd])
    g.add("attn_o", "library_call", ["ctx_r", "Wo"], [T, Hd], callee="matmul")
    for p in ("b_o", "g1", "be1"):
        g.param(p, [Hd])
    g.param("dmask_o", [T, Hd])
    g.add("b_o_b", "broadcast", ["b_o"], [T, Hd], broadcast_dim_map=[1])
    g.add("attn_ob", "add", ["attn_o", "b_o_b"], [T, Hd])
    g.add("attn_od", "mul", ["attn_ob", "dmask_o"], [T, Hd])
    g.add("res1", "add", ["attn_od", "x"], [T, Hd])
    _layernorm(g, "res1", "g1", "be1", T, Hd, "ln1.", "h1")
    g.param("W1", [Hd, FF])
    g.param("b_f1", [FF])
    g.add("ff1", "library_call", ["h1", "W1"], [T, FF], callee="matmul")
    g.add("b_f1_b", "broadcast", ["b_f1"], [T, FF], broadcast_dim_map=[1])
    g.add("u", "add", ["ff1", "b_f1_b"], [T, FF])
    g.add("u2", "mul", ["u", "u"], [T, FF])
    g.add("u3", "mul", ["u2", "u"], [T, FF])
    g.add("u3s", "scale", ["u3"], [T, FF], scalar=0.044715)
    g.add("inner", "add", ["u", "u3s"], [T, FF])
    g.add("inner_s", "scale", ["inner"], [T, FF], scalar=0.7978845608028654)
    g.add("th", "tanh", ["inner_s"], [T, FF])
    g.add("one", "constant", [], [T, FF], value=1.0)
    g.add("th1", "add", ["th", "one"], [T, FF])
    g.add("half_u", "scale", ["u"], [T, FF], scalar=0.5)
    g.add("gelu", "mul", ["half_u", "th1"], [T, FF])
    g.param("W2", [FF, Hd])
    g.add("ff2", "library_call", ["gelu", "W2"], [T, Hd], callee="matmul")
    for p in ("b_f2", "g2", "be2"):
        g.param(p, [Hd])
    g.param("dmask_f", [T, Hd])
    g.add("b_f2_b", "broadcast", ["b_f2"], [T, Hd], broadcast_dim_map=[1])
    g.add("ff2b", "add", ["ff2", "b_f2_b"], [T, Hd])
    g.add("ff2d", "mul", ["ff2b", "dmask_f"], [T, Hd])
    g.add("res2", "add", ["ff2d", "h1"], [T, Hd])
    _layernorm(g, "res2", "g2", "be2", T, Hd, "ln2.", "h2")
    return g.doc(["h2"])


BUILDERS = {
    "C1": c1_layernorm,
    "C2": c2_softmax,
    "C3": c3_biasgrad,
    "C3b": lambda **k: c3_biasgrad(with_dx=True, **k),
    "C4": c4_transpose,
    "C4b": c4b_transpose,
    "C4t": c4t_transpose,
    "C5": c5_bert,
    "C5L": c5_layer,
}

# Full sizes = BASELINE.json configs.  The small sizes are the CPU-oracle-sized
# parity cases (same graph structure, reference plan recomputed at that size).
FULL = {
    "C1": dict(R=8192, C=1024),
    "C2": dict(B=16, H=16, S=512, L=512),
    "C3": dict(N=65536, C=1024),
    "C3b": dict(N=65536, C=1024),
    "C4": dict(B=32, S=512, H=16, D=64),
    "C4b": dict(B=32, S=512, H=16, D=64),
    "C4t": dict(B=32, S=512, H=16, D=64),
    "C5": dict(B=64, S=512),
    "C5L": dict(B=64, S=512),
}

SMALL = {
    "C1": dict(R=64, C=1024),
    "C2": dict(B=2, H=2, S=16, L=512),
    "C3": dict(N=2048, C=1024),
    "C3b": dict(N=2048, C=1024),
    "C4": dict(B=2, S=64, H=16, D=64),
    "C4b": dict(B=2, S=64, H=16, D=64),
    "C4t": dict(B=2, S=64, H=16, D=64),
    "C5": dict(B=8, S=64),
    "C5L": dict(B=2, S=64),
}


def build(name: str, **sizes) -> dict:
    return BUILDERS[name](**sizes)


def dumps(doc: dict) -> str:
    return json.dumps(doc, indent=1) + "\n"


# Batch sharding: the dimension each config is split along
# across ranks, and the per-rank sizes of an n-way shard.  Rank r owns
# indices [r*N/n, (r+1)*N/n) of that dimension; every other size is unchanged.
SHARD_DIM = {"C1": "R", "C2": "B", "C3": "N", "C3b": "N", "C4": "B", "C4b": "B", "C4t": "B", "C5": "B", "C5L": "B"}
SHARD_COUNTS = (2, 4, 8)


def shard_sizes(name: str, n: int) -> dict:
    sizes = dict(FULL[name])
    d = SHARD_DIM[name]
    if sizes[d] % n:
        raise ValueError(f"{name}: {d}={sizes[d]} does not split {n} ways")
    sizes[d] //= n
    return sizes

