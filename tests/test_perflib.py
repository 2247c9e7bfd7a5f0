"""Measured B200 performance library (tools/measure_perflib.py output, committed
in workloads/perflib/) in the reference's text format (tuning.cpp:41-125):
well-formed, non-synthetic, keyed like make_perf_key (tuning.cpp:154-167) on the
plan's scheduled members, and — when the reference tool is built here —
accepted by the reference's own PerfLibrary parser and planner."""

import json
import os
import re
import subprocess

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
