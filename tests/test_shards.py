"""Batch-sharded plans: rank r of n runs the reference's plan of
its shard graph (the named config with the shard dimension divided by n).

The reference planner's 64 MiB footprint cap makes group membership
size-dependent (fusion.cpp:69-85; C5 merges h1+h2 into one group at B <= 7),
so a shard plan is only valid for the sharded benchmark if its membership,
roots and kernel count equal the global plan's.  Checked for every committed
shard plan (exported by the reference's own compile_graph via ref_tool)."""

import json
import os

import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H
from workloads import configs


def _membership(bundle):
    return ([(k["fusion_root"], sorted(k["members"]), list(k["roots"])) for k in bundle["kernels"]],
            sorted(bundle.get("unfused", [])), bundle["fused_kernels"])


CASES = [(c, n) for c in configs.SHARD_DIM if c != "C5L" for n in configs.SHARD_COUNTS]


@pytest.mark.parametrize("name,n", CASES)
def test_shard_plan_membership_equals_global_plan(name, n):
    with open(os.path.join(T.PLANS, f"{name}.full.json")) as f:
        full = json.load(f)
    with open(os.path.join(T.PLANS, f"{name}.shard{n}.json")) as f:
        shard = json.load(f)
    assert shard["workload"]["sizes"] == configs.shard_sizes(name, n)
    assert _membership(shard) == _membership(full)
    # the shard graph is the global graph with the shard dimension divided by n
    gs, gf = H.graph_from_json(shard["graph"]), H.graph_from_json(full["graph"])
    assert [i.id for i in gs.instructions] == [i.id for i in gf.instructions]
    assert sum(i.numel() for i in gs.parameters()) * n >= sum(i.numel() for i in gf.parameters())
    for a, b in zip(gs.parameters(), gf.parameters()):
        assert a.numel() in (b.numel(), b.numel() // n), a.id


@pytest.mark.skipif(not T.have_ref_tool(), reason="reference tool not built (no /root/reference here)")
@pytest.mark.parametrize("n", [2, 4, 8])
def test_shard_plans_are_the_references_plans(n):
    """Re-planned live by the reference (build container): the committed C5
    shard plan is exactly its compile_graph output."""
    from workloads.make_workloads import plan_bundle
    b = plan_bundle(configs.build("C5", **configs.shard_sizes("C5", n)))
    with open(os.path.join(T.PLANS, f"C5.shard{n}.json")) as f:
        want = json.load(f)
    assert _membership(b) == _membership(want)
    assert [k["statements"] for k in b["kernels"]] == [k["statements"] for k in want["kernels"]]


@pytest.mark.skipif(not T.have_ref_tool(), reason="reference tool not built (no /root/reference here)")
def test_membership_is_size_dependent():
    """Why the check matters: at b7 s512 the reference merges C5's two LayerNorm
    groups (4 groups), so 16 ranks over b64 (b4 each) would not run the global plan."""
    from workloads.make_workloads import plan_bundle
    assert len(plan_bundle(configs.build("C5", B=8, S=512))["kernels"]) == 5
    assert len(plan_bundle(configs.build("C5", B=7, S=512))["kernels"]) == 4
