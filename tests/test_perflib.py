"""Measured B200 performance library (tools/measure_perflib.py output, committed
in workloads/perflib/) in the reference's text format (tuning.cpp:41-125):
well-formed, non-synthetic, keyed like make_perf_key (tuning.cpp:154-167) on the
plan's scheduled members, and — when the reference tool is built here —
accepted by the reference's own PerfLibrary parser and planner."""

import json
import os
import re
import subprocess
import sys

import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H

LIBS = os.path.join(T.ROOT, "workloads", "perflib")
CONFIGS = ["C1", "C2", "C3", "C4", "C5"]
LINE = re.compile(r"^[a-z_]+\|[0-9,]*\|\d+\|\d+\|(row|col)\|\d+\|(-|\d+)\|[0-9.e+-]+\|0$")


@pytest.mark.parametrize("cfg", CONFIGS)
def test_perflib_format_and_keys(cfg):
    lines = [l.rstrip("\n") for l in open(os.path.join(LIBS, f"{cfg}.b200.lib")) if not l.startswith("#")]
    assert lines and all(LINE.match(l) for l in lines), lines[:3]
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, f"{cfg}.full.json"))
    keys = {"|".join(l.split("|")[:7]) for l in lines}
    for k in b["kernels"]:
        for m, (sd, sw, st) in k["per_instruction"].items():
            ins = g.at(m)
            extra = str(k["block_threads"] // 32) if ins.op in ("reduce", "transpose") else "-"
            key = "|".join([ins.op, ",".join(map(str, ins.shape)), str(sd), str(sw), st, str(k["block_threads"]), extra])
            assert key in keys, key


@pytest.mark.skipif(not T.have_ref_tool(), reason="reference tool not built here")
@pytest.mark.parametrize("cfg", CONFIGS)
def test_reference_planner_consumes_measured_library(cfg):
    out = subprocess.run([T.REF_TOOL, "perflib", os.path.join(T.PLANS, f"{cfg}.full.json"),
                          os.path.join(LIBS, f"{cfg}.b200.lib")], capture_output=True, text=True, check=True)
    d = json.loads(out.stdout)
    assert d["measured_entries"] > 0 and d["hits"] > 0
    assert d["fused_kernels"] == d["fused_kernels_default"]
    assert all(k["same_members_as_default"] for k in d["kernels"])
    header = open(os.path.join(LIBS, f"{cfg}.b200.lib")).readline()
    assert "NVIDIA B200" in header
    # chosen plans now cost the measured device time (microseconds, not the synthetic 500 GB/s model)
    assert all(k["cost_us"] < 1000 for k in d["kernels"])


DEVICE_PARITY = os.path.join(T.ROOT, "oracle", "_ref", "device_parity")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEVICE_PARITY), reason="reference harness not built (needs /root/reference)")
@pytest.mark.parametrize("name,sizes", [("C1", dict(R=64, C=1024)), ("C4", dict(B=2, S=64, H=16, D=64))])
def test_perflib_misses_measured_on_device(tmp_path, name, sizes):
    """The paper's library-miss path on the B200, through the
    reference-side binding: every perf key the reference planner misses is timed
    on the device (the instruction alone, literal tier, under that key's
    schedule and block size) and recorded non-synthetic in the reference's own
    format; re-planning then misses nothing.  The planned groups' template
    parameters are measured on miss into the template cache (a second pass hits
    everything), and a fresh process lowering with that cache uses them."""
    from workloads import configs
    graph = tmp_path / "g.json"
    graph.write_text(configs.dumps(configs.build(name, **sizes)))
    lib, tp = tmp_path / "measured.lib", tmp_path / "template_params.txt"
    env = dict(os.environ, SFX_TEMPLATE_PARAMS=str(tmp_path / "none.txt"))
    r = subprocess.run([DEVICE_PARITY, "perflib", str(graph), str(lib), str(tp)], capture_output=True, text=True,
                       timeout=1500, env=env)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0, d
    assert d["keys_measured"] == d["keys_missed"] > 0 and d["replan_misses"] == 0
    assert d["groups_tuned"] >= 1 and d["retune_groups_tuned"] == 0
    # the stored library parses with the reference's format: every entry measured
    entries = [l for l in open(lib) if l.strip() and not l.startswith("#")]
    assert len(entries) == d["measured_entries"] and all(l.rstrip().endswith("|0") for l in entries)
    # the template cache round-trips: a new process lowering with it finds every group
    tpl = [l for l in open(tp) if not l.startswith("#")]
    assert len(tpl) == d["groups_tuned"]
    g = H.graph_from_json(json.loads(graph.read_text()))
    bundle = json.loads(subprocess.run([T.REF_TOOL, "plan", str(graph)], capture_output=True, text=True).stdout) \
        if os.path.exists(T.REF_TOOL) else None
    if bundle is not None:
        code = ("import sys, json; sys.path.insert(0, %r); import paper_1811_05213_b200 as P; "
                "b = json.load(open(%r)); g = P.graph_from_json(b['graph']); r = P.CompileReport.from_bundle(b); "
                "print('\\n'.join(P.codegen(g, k.program)[2] for k in r.kernels))") % (T.ROOT, str(tmp_path / "b.json"))
        (tmp_path / "b.json").write_text(json.dumps(bundle))
        notes = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                               env=dict(os.environ, SFX_TEMPLATE_PARAMS=str(tp))).stdout.splitlines()
        assert sum("[template_params:" in n for n in notes) == d["groups_tuned"], notes
