"""Reference plans for extra parity shapes beyond BASELINE.json (long rows that
need the multi-warp row template, odd row counts), exported by the reference's
own compile_graph via oracle/_ref/ref_tool.  Build container only.

    python tests/golden/make_extra_plans.py
"""

import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from workloads import configs  # noqa: E402

def bn_graph(shape, rdims, with_stats=False, count=None):
    """Batch-norm statistics + normalise over `rdims` (contiguous), gamma/beta on
    the kept dims.  `count`: the number of reduced elements the means divide by
    — a rank's shard of a SyncBatchNorm graph divides by the GLOBAL count (explicit
    sum + scale instead of the parser's mean lowering, ir.cpp:396-428)."""
    kept = [d for d in range(len(shape)) if d not in rdims]
    cshape = [shape[d] for d in kept]

    def mean(name, src):
        if count is None:
            return [{"id": name, "op": "reduce", "operands": [src], "shape": cshape, "reduce_dims": rdims,
                     "reducer": "mean"}]
        return [{"id": name + ".sum", "op": "reduce", "operands": [src], "shape": cshape, "reduce_dims": rdims,
                 "reducer": "sum"},
                {"id": name, "op": "scale", "operands": [name + ".sum"], "shape": cshape, "scalar": 1.0 / count}]
    ins = [
        {"id": "x", "op": "parameter", "shape": shape},
        {"id": "g", "op": "parameter", "shape": cshape},
        {"id": "b", "op": "parameter", "shape": cshape}] + mean("mean", "x") + [
        {"id": "mean_b", "op": "broadcast", "operands": ["mean"], "shape": shape, "broadcast_dim_map": kept},
        {"id": "d", "op": "sub", "operands": ["x", "mean_b"], "shape": shape},
        {"id": "d2", "op": "mul", "operands": ["d", "d"], "shape": shape}] + mean("var", "d2") + [
        {"id": "eps", "op": "constant", "shape": cshape, "value": 1e-5},
        {"id": "ve", "op": "add", "operands": ["var", "eps"], "shape": cshape},
        {"id": "rstd", "op": "rsqrt", "operands": ["ve"], "shape": cshape},
        {"id": "rstd_b", "op": "broadcast", "operands": ["rstd"], "shape": shape, "broadcast_dim_map": kept},
        {"id": "n", "op": "mul", "operands": ["d", "rstd_b"], "shape": shape},
        {"id": "g_b", "op": "broadcast", "operands": ["g"], "shape": shape, "broadcast_dim_map": kept},
        {"id": "b_b", "op": "broadcast", "operands": ["b"], "shape": shape, "broadcast_dim_map": kept},
        {"id": "ng", "op": "mul", "operands": ["n", "g_b"], "shape": shape},
        {"id": "y", "op": "add", "operands": ["ng", "b_b"], "shape": shape}]
    outs = ["y"]
    if with_stats:
        ins.append({"id": "rstd_out", "op": "scale", "operands": ["rstd"], "shape": cshape, "scalar": 1.0})
        outs.append("rstd_out")
    return {"instructions": ins, "outputs": outs}


EXTRA = {
    "ln_r64_c8192": configs.c1_layernorm(R=64, C=8192),
    "ln_r100_c3072": configs.c1_layernorm(R=100, C=3072),
    "ln_r37_c2048": configs.c1_layernorm(R=37, C=2048),
    "softmax_r16_c16384": configs.c2_softmax(B=1, H=2, S=8, L=16384),
    "softmax_r24_c4096": configs.c2_softmax(B=2, H=3, S=4, L=4096),
    # rows beyond the register-resident template: one CTA per row, multi-pass
    "softmax_r4_c131072": configs.c2_softmax(B=1, H=1, S=4, L=131072),
    "softmax_r8_c131072": configs.c2_softmax(B=1, H=1, S=8, L=131072),  # special-value long softmax rows
    "softmax_r2_c262144": configs.c2_softmax(B=1, H=1, S=2, L=262144),  # 16-CTA (non-portable) cluster
    "ln_r6_c98304": configs.c1_layernorm(R=6, C=98304),
    "ln_r5_c70001": configs.c1_layernorm(R=5, C=70001),
    # more rows than persistent clusters (row_pipeline=3 loops rows per cluster)
    "softmax_r40_c131072": configs.c2_softmax(B=1, H=1, S=40, L=131072),
    
    # a single-reduction group (RMSNorm: one reduce level + element roots)
    "rms_r80_c98304": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [80, 98304]},
        {"id": "g", "op": "parameter", "shape": [98304]},
        {"id": "x2", "op": "mul", "operands": ["x", "x"], "shape": [80, 98304]},
        {"id": "ms", "op": "reduce", "operands": ["x2"], "shape": [80], "reduce_dims": [1], "reducer": "mean"},
        {"id": "eps", "op": "constant", "shape": [80], "value": 1e-6},
        {"id": "mse", "op": "add", "operands": ["ms", "eps"], "shape": [80]},
        {"id": "r", "op": "rsqrt", "operands": ["mse"], "shape": [80]},
        {"id": "rb", "op": "broadcast", "operands": ["r"], "shape": [80, 98304], "broadcast_dim_map": [0]},
        {"id": "gb", "op": "broadcast", "operands": ["g"], "shape": [80, 98304], "broadcast_dim_map": [1]},
        {"id": "n", "op": "mul", "operands": ["x", "rb"], "shape": [80, 98304]},
        {"id": "y", "op": "mul", "operands": ["n", "gb"], "shape": [80, 98304]}], "outputs": ["y"]},
    # masked softmax over long rows with e also output (2e): two staged inputs, the
    # cached member e (written over x's slice) feeds two roots of the final pass
    "softmaxmask_r4_c131072": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [4, 131072]},
        {"id": "mask", "op": "parameter", "shape": [4, 131072]},
        {"id": "xm", "op": "add", "operands": ["x", "mask"], "shape": [4, 131072]},
        {"id": "mx", "op": "reduce", "operands": ["xm"], "shape": [4], "reduce_dims": [1], "reducer": "max"},
        {"id": "mxb", "op": "broadcast", "operands": ["mx"], "shape": [4, 131072], "broadcast_dim_map": [0]},
        {"id": "z", "op": "sub", "operands": ["xm", "mxb"], "shape": [4, 131072]},
        {"id": "e", "op": "exp", "operands": ["z"], "shape": [4, 131072]},
        {"id": "s", "op": "reduce", "operands": ["e"], "shape": [4], "reduce_dims": [1], "reducer": "sum"},
        {"id": "sb", "op": "broadcast", "operands": ["s"], "shape": [4, 131072], "broadcast_dim_map": [0]},
        {"id": "y", "op": "div", "operands": ["e", "sb"], "shape": [4, 131072]},
        {"id": "e_out", "op": "scale", "operands": ["e"], "shape": [4, 131072], "scalar": 2.0}], "outputs": ["y", "e_out"]},
    # batch-norm backward-like: two column sums of two streamed inputs (dy, x)
    # broadcast back — the colbc cp.async ring with two staged inputs
    "bnbwd_4096x256": {"instructions": [
        {"id": "dy", "op": "parameter", "shape": [4096, 256]},
        {"id": "x", "op": "parameter", "shape": [4096, 256]},
        {"id": "s1", "op": "reduce", "operands": ["dy"], "shape": [256], "reduce_dims": [0], "reducer": "sum"},
        {"id": "dyx", "op": "mul", "operands": ["dy", "x"], "shape": [4096, 256]},
        {"id": "s2", "op": "reduce", "operands": ["dyx"], "shape": [256], "reduce_dims": [0], "reducer": "sum"},
        {"id": "m1", "op": "scale", "operands": ["s1"], "shape": [256], "scalar": 1.0 / 4096},
        {"id": "m2", "op": "scale", "operands": ["s2"], "shape": [256], "scalar": 1.0 / 4096},
        {"id": "m1b", "op": "broadcast", "operands": ["m1"], "shape": [4096, 256], "broadcast_dim_map": [1]},
        {"id": "m2b", "op": "broadcast", "operands": ["m2"], "shape": [4096, 256], "broadcast_dim_map": [1]},
        {"id": "t1", "op": "sub", "operands": ["dy", "m1b"], "shape": [4096, 256]},
        {"id": "t2", "op": "mul", "operands": ["x", "m2b"], "shape": [4096, 256]},
        {"id": "dx", "op": "sub", "operands": ["t1", "t2"], "shape": [4096, 256]}], "outputs": ["dx"]},
    # innermost-moving transposes with ragged 64x64 tiles: the 128-bit swizzled
    # tile (both axes multiples of 4) and the scalar tile (odd extents)
    "tr_8x300x140": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [8, 300, 140]},
        {"id": "b", "op": "parameter", "shape": [140]},
        {"id": "bb", "op": "broadcast", "operands": ["b"], "shape": [8, 300, 140], "broadcast_dim_map": [2]},
        {"id": "xb", "op": "add", "operands": ["x", "bb"], "shape": [8, 300, 140]},
        {"id": "xt", "op": "transpose", "operands": ["xb"], "shape": [8, 140, 300], "permutation": [0, 2, 1]},
        {"id": "y", "op": "scale", "operands": ["xt"], "shape": [8, 140, 300], "scalar": 0.125}], "outputs": ["y"]},
    "tr_8x301x141": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [8, 301, 141]},
        {"id": "xt", "op": "transpose", "operands": ["x"], "shape": [8, 141, 301], "permutation": [0, 2, 1]},
        {"id": "y", "op": "exp", "operands": ["xt"], "shape": [8, 141, 301]}], "outputs": ["y"]},
    # column statistics broadcast back (batch-norm): the colbc template
    "bn_4096x256": bn_graph([4096, 256], [0]),
    "bn_mid_8x512x64": bn_graph([8, 512, 64], [1]),
    "bn_nhwc_16x16x8x128": bn_graph([16, 16, 8, 128], [0, 1, 2], with_stats=True),
    # batch-norm over NCHW: reduced dims on both sides of the channel block
    # ([A | K | B]); the reference plans it as one group of one block
    "bn_nchw_16x8x64x64": bn_graph([16, 8, 64, 64], [0, 2, 3]),  # 16 stripes per channel: grid barrier
    "bn_nchw_4x160x7x7": bn_graph([4, 160, 7, 7], [0, 2, 3]),  # B = 49: scalar vectors
    "bn_nchw_8x32x14x14": bn_graph([8, 32, 14, 14], [0, 2, 3], with_stats=True),  # channel root
    "bn_nchw_8x80x64x64": bn_graph([8, 80, 64, 64], [0, 2, 3], with_stats=True),  # clusters of 8 CTAs per channel
    "bn_nchw_8x96x32x32": bn_graph([8, 96, 32, 32], [0, 2, 3]),  # clusters of 2
    # one rank"s shard of a 2-rank SyncBatchNorm over 4096 rows (global count)
    "bnsync_shard_2048x256": bn_graph([2048, 256], [0], count=4096),
    "bnmax_3000x37": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [3000, 37]},
        {"id": "m", "op": "reduce", "operands": ["x"], "shape": [37], "reduce_dims": [0], "reducer": "max"},
        {"id": "mb", "op": "broadcast", "operands": ["m"], "shape": [3000, 37], "broadcast_dim_map": [1]},
        {"id": "z", "op": "sub", "operands": ["x", "mb"], "shape": [3000, 37]},
        {"id": "e", "op": "exp", "operands": ["z"], "shape": [3000, 37]}], "outputs": ["e"]},
    # middle-axis and full reductions: the [outer | reduced | inner] column template
    "midsum_16x4096x64": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [16, 4096, 64]},
        {"id": "e", "op": "exp", "operands": ["x"], "shape": [16, 4096, 64]},
        {"id": "s", "op": "reduce", "operands": ["e"], "shape": [16, 64], "reduce_dims": [1], "reducer": "sum"},
        {"id": "y", "op": "scale", "operands": ["s"], "shape": [16, 64], "scalar": 0.5}], "outputs": ["y"]},
    "midmax_7x999x3_i32": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [7, 999, 3], "dtype": "i32"},
        {"id": "n", "op": "neg", "operands": ["x"], "shape": [7, 999, 3], "dtype": "i32"},
        {"id": "m", "op": "reduce", "operands": ["n"], "shape": [7, 3], "reduce_dims": [1], "reducer": "max",
         "dtype": "i32"}], "outputs": ["m"]},
    "fullmax_1024x1000": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [1024, 1000]},
        {"id": "m", "op": "reduce", "operands": ["x"], "shape": [], "reduce_dims": [0, 1], "reducer": "max"},
        {"id": "y", "op": "neg", "operands": ["m"], "shape": []}], "outputs": ["y"]},
    "fullsum_3x5000x7": {"instructions": [
        {"id": "x", "op": "parameter", "shape": [3, 5000, 7]},
        {"id": "t", "op": "tanh", "operands": ["x"], "shape": [3, 5000, 7]},
        {"id": "s", "op": "reduce", "operands": ["t"], "shape": [], "reduce_dims": [0, 1, 2], "reducer": "sum"}],
        "outputs": ["s"]},
}


def two_cross_rank_groups(rows=2048, cols=256, count=4096):
    """One rank's shard with TWO independent batch-crossing groups: SyncBatchNorm
    over x (colbc) and a bias-grad column sum over (dy, z) (col).  Both wait on
    the peer ranks inside the kernel, so the executor must run them in the same
    order on every rank (never on parallel branches)."""
    bn = bn_graph([rows, cols], [0], count=count)
    ins = bn["instructions"] + [
        {"id": "dy", "op": "parameter", "shape": [rows, cols]},
        {"id": "z", "op": "parameter", "shape": [rows, cols]},
        {"id": "zero", "op": "constant", "shape": [rows, cols], "value": 0.0},
        {"id": "mask", "op": "compare", "operands": ["z", "zero"], "shape": [rows, cols]},
        {"id": "dx", "op": "mul", "operands": ["dy", "mask"], "shape": [rows, cols]},
        {"id": "db", "op": "reduce", "operands": ["dx"], "shape": [cols], "reduce_dims": [0], "reducer": "sum"}]
    return {"instructions": ins, "outputs": ["y", "db"]}


# batch-sharded graphs run with cross_rank (tests/test_gpu_peer.py)
XRANK = {"two_xrank_shard_2048x256": two_cross_rank_groups()}


def fixture_plans():
    """The reference's own fixture graphs (tests/golden/fixtures, fixtures.cpp)
    as planned by its tests: softmax_batchdot with fuse_dot (test_exec.cpp:157-174),
    elementwise_chain with default options (:176-194)."""
    fix = os.path.join(HERE, "fixtures")
    return {"softmax_batchdot_fusedot": (json.load(open(os.path.join(fix, "softmax_batchdot.json"))), ["--fuse-dot"]),
            "elementwise_chain": (json.load(open(os.path.join(fix, "elementwise_chain.json"))), [])}


def main():
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    for sub, table in (("plans_extra", EXTRA), ("plans_xrank", XRANK), ("plans_fixtures", fixture_plans())):
        export(tool, os.path.join(HERE, sub), table)


def export(tool, out_dir, table):
    os.makedirs(out_dir, exist_ok=True)
    for name, doc in table.items():
        flags = []
        if isinstance(doc, tuple):
            doc, flags = doc
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            f.write(configs.dumps(doc))
            path = f.name
        try:
            out = subprocess.run([tool, "plan", path] + flags, check=True, capture_output=True, text=True).stdout
        finally:
            os.unlink(path)
        b = json.loads(out)
        for k in b["kernels"]:
            k.pop("dump", None)
        with open(os.path.join(out_dir, name + ".json"), "w") as f:
            json.dump(b, f, separators=(",", ":"))
        print(name, b["fused_kernels"])


if __name__ == "__main__":
    main()
