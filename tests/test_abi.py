"""CPU-side checks of the product boundary: libsfx.so loads without a GPU,
exports every symbol include/sfx.h declares, rejects what the reference
rejects, and every committed reference plan lowers to CUDA that NVRTC compiles
to sm_100a SASS (no GPU needed for that)."""

import os

import numpy as np
import re
import subprocess

import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H

HEADER = os.path.join(T.ROOT, "include", "sfx.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:sfx_status|int32_t|int64_t|const char\*)\s+(sfx_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = H.lib()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(H.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", H.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sfx_\w+)", out))
    assert set(names) <= exported
    assert L.sfx_abi_version() == H.ABI_VERSION == 3


def test_ctx_create_without_gpu_fails_loudly():
    import ctypes as C
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = H.lib().sfx_ctx_create(0, C.byref(h))
    assert st == 4  # SFX_ERR_CUDA
    assert b"libcuda" in H.lib().sfx_last_error() or b"cuInit" in H.lib().sfx_last_error()


WORKLOADS = sorted(f[:-5] for f in os.listdir(T.PLANS) if f.endswith(".json"))

EXPECTED = {  # strategy the GroupAnalyzer must pick at full size
    ("C1", "y"): "row", ("C2", "y"): "row", ("C3", "db"): "col", ("C3b", "db"): "col",
    ("C3b", "dx_out"): "map", ("C4", "y"): "map", ("C4b", "y"): "map", ("C4t", "y"): "map", ("C5", "ctx_r"): "map",
    ("C5", "gelu"): "map", ("C5", "h1"): "row", ("C5", "h2"): "row", ("C5", "probs_d"): "row",
    ("C5L", "h2"): "row", ("C5L", "gelu"): "map", ("C5L", "h1"): "row", ("C5L", "ctx_r"): "map",
    ("C5L", "probs_d"): "map", ("C5L", "v_t"): "map", ("C5L", "sm.e"): "row", ("C5L", "k_t"): "map",
    ("C5L", "q_t"): "map",
    # C5L planned with fuse_dot: the attention matmuls stitched with their operand producers
    ("C5LF", "h2"): "row", ("C5LF", "gelu"): "map", ("C5LF", "h1"): "row", ("C5LF", "ctx_r"): "map",
    ("C5LF", "ctx"): "dot", ("C5LF", "sm.e"): "row", ("C5LF", "scores"): "dot",
}


@pytest.mark.parametrize("wl", WORKLOADS)
def test_workload_plans_lower_and_compile_for_sm100a(wl):
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, wl + ".json"))
    name, size = wl.split(".")
    unfused = T.unfused_kernels(g, rep)
    assert len(rep.kernels) + sum(g.at(u).op != "library_call" for u in unfused) == b["fused_kernels"]
    for k in rep.kernels:
        for strategy in ("auto", "literal"):
            src, cubin, note = H.codegen(g, k.program, strategy)
            assert os.path.getsize(cubin) > 0
            assert "extern \"C\" __global__" in src
            if strategy == "auto" and size == "full":
                assert note.split()[0] == EXPECTED[(name, k.program.fusion_root)], note
    for i, u in enumerate(unfused):
        src, cubin, note = H.codegen_barrier(g, rep, i)
        assert os.path.getsize(cubin) > 0
        if g.at(u).op in ("batch_matmul", "library_call"):
            assert note.startswith("dot"), note


def test_full_size_streams_are_128bit():
    """The map/row/col kernels on the named shapes move HBM data with LDG.E.128 / STG.E.128."""
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C5.full.json"))
    for k in rep.kernels:
        src, cubin, note = H.codegen(g, k.program)
        sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
        assert re.search(r"LDG\.E(\.\w+)*\.128", sass), k.program.fusion_root
        assert re.search(r"STG\.E(\.\w+)*\.128", sass), k.program.fusion_root


def _eligible(stream, limit=None):
    d = T.load_json(os.path.join(T.GOLDEN, f"random_{stream}.json"))
    out = [c for c in d["cases"] if c["device_eligible"]]
    return out[:limit] if limit else out


def test_random_graph_groups_lower_and_compile():
    """Every group of the device-eligible reference random graphs compiles in both tiers."""
    n = 0
    for case in _eligible("pipeline"):
        g = H.graph_from_json(case["bundle"]["graph"])
        rep = H.CompileReport.from_bundle(case["bundle"])
        for k in rep.kernels:
            for strategy in ("auto", "literal"):
                H.codegen(g, k.program, strategy)
                n += 1
    assert n > 40


def test_matmul_groups_lower():
    """fuse_dot groups: a lone BatchMatMul uses the dot kernel; a BatchMatMul that
    is the group's only root, stitched to elementwise / layout members producing
    its operands, the dot kernel with those members computed where its tiles are
    staged ("fuse_dot group"); anything else (reductions feeding it, other roots)
    the literal tier (dot_loop in reference k order)."""
    d = T.load_json(os.path.join(T.GOLDEN, "random_acceptance.json"))
    seen = set()
    for case in d["cases"]:
        if not case["bundle"]["options"]["fuse_dot"]:
            continue
        g = H.graph_from_json(case["bundle"]["graph"])
        rep = H.CompileReport.from_bundle(case["bundle"])
        for k in rep.kernels:
            if not any(g.at(m).op == "batch_matmul" for m in k.program.members):
                continue
            _, cubin, note = H.codegen(g, k.program)
            members = [g.at(m) for m in k.program.members]
            dots = [m for m in members if m.op == "batch_matmul"]
            prologue = (len(dots) == 1 and list(k.program.roots) == [dots[0].id] and
                        all(m.op in ("batch_matmul", "reshape", "bitcast", "transpose", "broadcast") or
                            m.op not in ("reduce", "library_call", "parameter", "constant") for m in members) and
                        not any(m.op == "reduce" and int(np.prod(m.shape or [1])) != int(np.prod(g.at(m.operands[0]).shape or [1]))
                                for m in members))
            kind = "dot" if len(members) == 1 else "dotp" if prologue else "literal"
            if kind == "dotp":
                assert note.startswith("dot fuse_dot group"), note
            else:
                assert note.split()[0] == kind, note
            seen.add(kind)
    assert seen == {"dot", "dotp", "literal"}, seen


def _assert_no_contraction(sass):
    """Every multiply-add of the dot kernel rounds twice: FMUL + FADD, or the
    packed FFMA2 whose addend is the same run-time zero pair in every
    instruction (the product alone) followed by FADD2; never a scalar FFMA."""
    import re
    lines = [l for l in sass.splitlines() if re.search(r"\bFFMA2?\b", l)]
    assert not [l for l in lines if re.search(r"\bFFMA\b", l)], "scalar FFMA contracts a multiply-add"
    addends = {re.split(r",\s*", l.split("FFMA2", 1)[1].split(";")[0])[-1].split(".")[0].strip() for l in lines}
    if lines:
        assert len(addends) == 1 and "FADD2" in sass, addends
    else:
        assert "FMUL" in sass and "FADD" in sass


def test_unfused_instructions_lower():
    """Instructions no group took (run by the reference through eval_dense)
    compile to one kernel each; matmuls to the dot kernel, whose fp32 loop has
    no FFMA (two roundings per step, as matmul_element, exec.cpp:84-100)."""
    n = {"dot": 0, "other": 0}
    for stream in ("pipeline", "acceptance"):
        d = T.load_json(os.path.join(T.GOLDEN, f"random_{stream}.json"))
        for case in d["cases"]:
            g = H.graph_from_json(case["bundle"]["graph"])
            rep = H.CompileReport.from_bundle(case["bundle"])
            for k, u in enumerate(T.unfused_kernels(g, rep)):
                src, cubin, note = H.codegen_barrier(g, rep, k)
                if g.at(u).op in ("batch_matmul", "library_call"):
                    assert note.startswith("dot matmul barrier"), note
                    if g.at(u).dtype == "f32" and n["dot"] < 8:
                        sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
                        _assert_no_contraction(sass)
                    n["dot"] += 1
                else:
                    n["other"] += 1
    assert n["dot"] >= 20 and n["other"] >= 1, n


def test_opaque_library_call_is_not_executable():
    g = H.graph_from_json({"instructions": [
        {"id": "a", "op": "parameter", "shape": [4, 8]},
        {"id": "b", "op": "parameter", "shape": [8, 2]},
        {"id": "c", "op": "library_call", "callee": "opaque", "operands": ["a", "b"], "shape": [4, 2]}],
        "outputs": ["c"]})
    rep = H.CompileReport([], 0, 0, 1.0, ["c"])
    with pytest.raises(H.ExecError) as e:  # exec.cpp:207-209
        H.codegen_barrier(g, rep, 0)
    assert e.value.status == 5 and "not executable" in str(e.value)


def test_malformed_program_is_rejected():
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C1.small.json"))
    p = rep.kernels[0].program
    bad = H.KernelProgram(p.fusion_root, p.members, p.roots, p.blocks, p.block_threads, p.arena_bytes,
                          [s for s in p.statements if s.get("dest") != "output"])
    with pytest.raises(H.ExecError) as e:
        H.codegen(g, bad)
    assert e.value.status == 1 and "not all roots written" in str(e.value)
    over = [dict(s) for s in p.statements]
    for s in over:
        if s.get("dest") == "shared":
            s["offset"] = p.arena_bytes
    with pytest.raises(H.ExecError) as e:
        H.codegen(g, H.KernelProgram(p.fusion_root, p.members, p.roots, p.blocks, p.block_threads,
                                     p.arena_bytes, over))
    assert "arena overflow" in str(e.value)


def test_forcing_an_inapplicable_template_fails():
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C3.small.json"))
    with pytest.raises(H.ExecError) as e:
        H.codegen(g, rep.kernels[0].program, "row")
    assert e.value.status == 2
    with pytest.raises(H.ExecError):
        H.codegen(g, rep.kernels[0].program, "map")


def test_parse_graph_lowers_mean_like_the_reference():
    from workloads import configs
    g = H.parse_graph(configs.dumps(configs.c1_layernorm(R=4, C=8)))
    gb, rep, b = H.load_bundle(os.path.join(T.PLANS, "C1.small.json"))
    assert [i.id for i in g.instructions] == [i.id for i in gb.instructions]
    assert g.at("ln.mean").op == "scale" and g.at("ln.mean").scalar == 1.0 / 8
    assert g.at("ln.mean.sum").op == "reduce"


def test_innermost_moving_transpose_uses_smem_tiles():
    """C4t (key transpose [B,S,H,D]->[B,H,D,S]) moves the innermost dimension:
    the map template stages it through a 64x64 shared-memory tile (XOR-swizzled
    128-bit rows here; the padded [64][65] scalar tile for odd extents)."""
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C4t.full.json"))
    src, cubin, note = H.codegen(g, rep.kernels[0].program)
    assert "smem-tiled" in note and "tile0[4096]" in src
    _, _, note1 = H.codegen(g, rep.kernels[0].program, row_pipeline=1)  # scalar tile (A/B knob)
    assert "XOR" not in note1
    sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
    assert "STS" in sass and "LDS" in sass and "BAR.SYNC" in sass


def test_cross_rank_rejects_non_column_batch_reduce():
    """A reduction over the sharded dim 0 that neither column template can take
    (reduce dims {0, 2}: not contiguous) fails loudly at compile time instead of
    silently reducing one shard.  (Column sums, and column statistics broadcast
    back — SyncBatchNorm — are combined across ranks in-kernel.)"""
    doc = {"instructions": [
        {"id": "p", "op": "parameter", "shape": [8, 16, 4]},
        {"id": "s", "op": "reduce", "operands": ["p"], "shape": [16], "reduce_dims": [0, 2], "reducer": "sum"},
        {"id": "y", "op": "scale", "operands": ["s"], "shape": [16], "scalar": 2.0},
    ], "outputs": ["y"]}
    g = H.graph_from_json(doc)
    prog = H.KernelProgram("y", ["s", "y"], ["y"], 1, 64, 64,
                           [{"kind": "materialize", "instr": "s", "schedule": [0, 1, "row"], "dest": "shared",
                             "offset": 0, "bytes": 64}, {"kind": "barrier"},
                            {"kind": "materialize", "instr": "y", "schedule": [0, 1, "row"], "dest": "output",
                             "root_index": 0}])
    with pytest.raises(H.ExecError, match="sharded dim 0"):
        H.codegen(g, prog, cross_rank=1)
    _, _, note = H.codegen(g, prog)  # single rank: the split column template takes it
    assert note.startswith("colbc split A=8 channels=16 B=4"), note


def test_cross_rank_accepts_sync_batchnorm():
    g, rep, _ = H.load_bundle(os.path.join(T.GOLDEN, "plans_extra", "bnsync_shard_2048x256.json"))
    src, _, note = H.codegen(g, rep.kernels[0].program, cross_rank=1)
    assert note.startswith("colbc") and "peers[p] + poff" in src and "launch_seq" in src


def test_ctypes_mirror_matches_c_struct_layout(tmp_path):
    """host.py's ctypes structures must match include/sfx.h field by field
    (sizes and offsets as the C compiler lays them out)."""
    import ctypes as C
    structs = {
        "sfx_instr": H.SfxInstr, "sfx_stmt": H.SfxStmt, "sfx_program": H.SfxProgram, "sfx_member_plan": H.SfxMemberPlan,
        "sfx_graph_desc": H.SfxGraphDesc, "sfx_compile_opts": H.SfxCompileOpts, "sfx_kernel_info": H.SfxKernelInfo,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sfx.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(T.ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                          check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} size"]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)
