"""The reference executor's self-checks (exec.cpp:320-327 stale arena read /
chunk containment, :399 overlapping root write, :410 incomplete coverage) on
the device path.  They depend only on the program's geometry, so libsfx.so
decides them when a program is handed in (csrc/ir.cpp
check_executor_geometry), with the reference's messages; these CPU tests feed
it the reference's own corrupted programs (test_exec.cpp:157-194) through the
codegen entry point, which needs no GPU."""

import copy
import json
import os

import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H

PLANS = os.path.join(T.GOLDEN, "plans_fixtures")


def _program(name):
    g, rep, _ = H.load_bundle(os.path.join(PLANS, name + ".json"))
    return g, copy.deepcopy(rep.kernels[0].program)


def test_valid_fixture_programs_pass():
    for name in ("softmax_batchdot_fusedot", "elementwise_chain"):
        g, prog = _program(name)
        H.codegen(g, prog)


def test_stale_arena_read_is_detected():
    """test_exec.cpp:157-174: divert the reduce writes to offset 0 while reads
    still target the mapped offsets (KernelProgram.arena_offsets)."""
    g, prog = _program("softmax_batchdot_fusedot")
    for st in prog.statements:
        if st["kind"] == "materialize" and st.get("dest") == "shared" and st["instr"] in ("Reduce.1", "Reduce.2"):
            st["offset"] = 0
    with pytest.raises(H.ExecError, match="stale arena read of "):
        H.codegen(g, prog)


def test_incomplete_coverage_is_detected():
    """test_exec.cpp:176-194: shrink the root chunk so blocks stop covering the output."""
    g, prog = _program("elementwise_chain")
    assert prog.blocks > 1
    for st in prog.statements:
        if st["kind"] == "materialize" and st.get("dest") == "output" and st["schedule"][1] > 1:
            st["schedule"] = [st["schedule"][0], st["schedule"][1] * 2, st["schedule"][2]]
    with pytest.raises(H.ExecError, match="incomplete coverage of root Chain.10"):
        H.codegen(g, prog)


def test_overlapping_root_write_is_detected():
    """Fewer boxes than blocks: later blocks repeat a box (exec.cpp:399)."""
    g, prog = _program("elementwise_chain")
    for st in prog.statements:
        if st["kind"] == "materialize" and st.get("dest") == "output":
            st["schedule"] = [st["schedule"][0], st["schedule"][1] // 2, st["schedule"][2]]
    with pytest.raises(H.ExecError, match="overlapping write to root Chain.10"):
        H.codegen(g, prog)


def test_chunk_containment_violation_is_detected():
    """A member read with a schedule (SchedulePlan.per_instruction) other than
    the one it was materialised with reads outside its chunk (exec.cpp:321-323)."""
    g, prog = _program("softmax_batchdot_fusedot")
    prog.per_instruction = dict(prog.per_instruction)
    sd, sw, ty = prog.per_instruction["Exponential.1"]
    prog.per_instruction["Exponential.1"] = [sd, sw * 2, ty]
    with pytest.raises(H.ExecError, match="chunk containment violation reading Exponential.1"):
        H.codegen(g, prog)
