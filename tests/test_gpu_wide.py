"""Tensors past 2^31 elements (8.6 GB each): the 64-bit index path of the map,
row and column templates (180 GB of HBM makes such groups realistic).  Inputs
are generated on the device; sampled rows / the column sums are checked against
an fp64 torch computation."""

import os

import numpy as np
import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H

WIDE = os.path.join(T.GOLDEN, "plans_wide")


@pytest.mark.parametrize("name,strategy", [("wide_map", "map"), ("wide_ln", "row"), ("wide_colsum", "col")])
def test_wide_codegen_uses_64bit_index(name, strategy):
    g, rep, _ = H.load_bundle(os.path.join(WIDE, name + ".json"))
    assert rep.fused_kernels == 1
    src, _, note = H.codegen(g, rep.kernels[0].program)
    assert note.startswith(strategy), note
    assert "long long" in src


@pytest.fixture(scope="module")
def env():
    import torch
    if torch.cuda.get_device_properties(0).total_memory < 40 * (1 << 30):
        pytest.skip("needs a large-memory GPU")
    ctx = H.Context(0)
    yield ctx, torch
    ctx.close()


def _kernel(ctx, name):
    g, rep, b = H.load_bundle(os.path.join(WIDE, name + ".json"))
    k = H.Kernel(ctx, g, rep.kernels[0].program)
    return g, k


@pytest.mark.gpu
def test_wide_map(env):
    ctx, torch = env
    g, k = _kernel(ctx, "wide_map")
    shape = g.at("x").shape
    assert g.at("x").numel() > 2 ** 31
    x = torch.rand(shape, device="cuda")
    y = torch.empty_like(x)
    k.launch([x.data_ptr()], [y.data_ptr()])
    torch.cuda.synchronize()
    for rows in (slice(0, 4), slice(shape[0] // 2, shape[0] // 2 + 4), slice(shape[0] - 4, shape[0])):
        want = (x[rows].double() * 0.5 + 1.0).float()
        assert torch.equal(y[rows], want)
    del x, y
    k.close()


@pytest.mark.gpu
def test_wide_layernorm_rows(env):
    ctx, torch = env
    g, k = _kernel(ctx, "wide_ln")
    R, C = g.at("x").shape
    x = torch.rand((R, C), device="cuda") * 2 - 1
    gamma = torch.rand(C, device="cuda")
    beta = torch.rand(C, device="cuda")
    y = torch.empty_like(x)
    ptr = {"x": x, "gamma": gamma, "beta": beta}
    k.launch([ptr[i].data_ptr() for i in k.input_ids], [y.data_ptr()])
    torch.cuda.synchronize()
    for r0 in (0, R // 2, R - 8):
        xs = x[r0:r0 + 8].double()
        mean = xs.mean(dim=1, keepdim=True)
        d = xs - mean
        var = (d * d).mean(dim=1, keepdim=True)
        want = (d / torch.sqrt(var + 1e-5) * gamma.double() + beta.double()).cpu().numpy()
        got = y[r0:r0 + 8].cpu().numpy()
        assert np.allclose(got, want, rtol=1e-5, atol=1e-6)
    del x, y
    k.close()


@pytest.mark.gpu
def test_wide_column_sum(env):
    ctx, torch = env
    g, k = _kernel(ctx, "wide_colsum")
    R, C = g.at("x").shape
    x = torch.rand((R, C), device="cuda") * 2 - 1
    s = torch.empty(C, device="cuda")
    k.launch([x.data_ptr()], [s.data_ptr()])
    torch.cuda.synchronize()
    want = x.double().sum(dim=0).cpu().numpy()
    got = s.cpu().numpy()
    assert np.allclose(got, want, rtol=1e-5, atol=1e-6 * np.sqrt(R))
    del x
    k.close()
