"""The packed-pair SIMT matmul (fma.rn.f32x2 with a run-time zero addend +
add.rn.f32x2) against the FMUL + FADD kernel and the reference's sequential fp32
loop (matmul_element, exec.cpp:84-100): bit for bit, on ragged tiles and on
signed zeros, subnormals, infinities and NaN."""

import os

import numpy as np
import pytest
import torch

import sfx_testlib as T  # noqa: F401
from paper_1811_05213_b200 import host as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = H.Context(0)
    yield c
    c.close()


def _matmul_graph(bd, M, K, N):
    ins = [{"id": "a", "op": "parameter", "shape": bd + [M, K]},
           {"id": "b", "op": "parameter", "shape": bd + [K, N]},
           {"id": "c", "op": "batch_matmul" if bd else "library_call", "operands": ["a", "b"], "shape": bd + [M, N]}]
    if not bd:
        ins[-1]["callee"] = "matmul"
    return H.graph_from_json({"instructions": ins, "outputs": ["c"]})


def _run(ctx, g, a, b, packed):
    old = os.environ.get("SFX_DOT_PACKED")
    os.environ["SFX_DOT_PACKED"] = "1" if packed else "0"
    try:
        cg = H.CompiledGraph(ctx, g, H.CompileReport([], 0, 0, 1.0, ["c"]))
    finally:
        if old is None:
            del os.environ["SFX_DOT_PACKED"]
        else:
            os.environ["SFX_DOT_PACKED"] = old
    try:
        note = cg.barrier_kernels[0].info["entry"], cg.barrier_kernels[0].info["smem_bytes"]
        c = torch.empty(list(a.shape[:-1]) + [b.shape[-1]], device="cuda")
        cg.run([a.data_ptr(), b.data_ptr()], [c.data_ptr()], stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        return c.cpu().numpy(), note
    finally:
        cg.close()


def _seq(A, B):
    """The reference's loop, vectorised over outputs: acc = fl(acc + fl(a*b)), k ascending."""
    acc = np.zeros((A.shape[0], B.shape[1]), np.float32)
    with np.errstate(all="ignore"):
        for k in range(A.shape[1]):
            acc = (acc + (A[:, k:k + 1] * B[k:k + 1, :]).astype(np.float32)).astype(np.float32)
    return acc


def _same_bits(x, y):
    xb, yb = x.view(np.uint32), y.view(np.uint32)
    nan = np.isnan(x) & np.isnan(y)
    return bool(np.all((xb == yb) | nan))


@pytest.mark.parametrize("bd,M,K,N", [([], 300, 100, 260), ([2], 256, 64, 384), ([], 129, 36, 132),
                                      ([4], 256, 128, 64), ([], 200, 40, 100)])  # last two: 128 x 64 tiles
def test_packed_matmul_bit_exact_ragged(ctx, bd, M, K, N):
    gen = torch.Generator(device="cuda").manual_seed(M + K + N)
    a = torch.rand(bd + [M, K], generator=gen, device="cuda") * 2 - 1
    b = torch.rand(bd + [K, N], generator=gen, device="cuda") * 2 - 1
    g = _matmul_graph(bd, M, K, N)
    cp, (ep, smem) = _run(ctx, g, a, b, True)
    cs, _ = _run(ctx, g, a, b, False)
    assert smem > 48 * 1024, "packed kernel (3-stage cp.async pipeline in dynamic shared memory) expected"
    assert _same_bits(cp, cs)
    A = a.reshape(-1, M, K).cpu().numpy()
    B = b.reshape(-1, K, N).cpu().numpy()
    C = cp.reshape(-1, M, N)
    for i in range(A.shape[0]):
        assert _same_bits(C[i], _seq(A[i], B[i]))


def test_packed_matmul_special_values(ctx):
    M, K, N = 256, 64, 256
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 2 ** 32, size=(M * K + K * N), dtype=np.uint64).astype(np.uint32)
    bits = (bits & np.uint32(0x8FFFFFFF)) | np.uint32(0x30000000)      # moderate magnitudes
    sel = rng.integers(0, 40, size=bits.shape)
    bits = np.where(sel == 0, np.uint32(0x80000000), bits)              # -0
    bits = np.where(sel == 1, np.uint32(0), bits)                       # +0
    bits = np.where(sel == 2, bits & np.uint32(0x807FFFFF), bits)       # subnormals
    bits = np.where(sel == 3, np.uint32(0x7F800000) | (bits & np.uint32(0x80000000)), bits)  # +-inf
    bits[7] = np.uint32(0x7FC00000)                                     # one NaN
    vals = bits.view(np.float32)
    a = torch.from_numpy(vals[:M * K].reshape(M, K).copy()).cuda()
    b = torch.from_numpy(vals[M * K:].reshape(K, N).copy()).cuda()
    g = _matmul_graph([], M, K, N)
    cp, _ = _run(ctx, g, a, b, True)
    cs, _ = _run(ctx, g, a, b, False)
    assert _same_bits(cp, cs)
    assert _same_bits(cp, _seq(a.cpu().numpy(), b.cpu().numpy()))
