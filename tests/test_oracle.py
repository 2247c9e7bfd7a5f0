"""The oracle restatement (oracle/sfx_oracle.c) pinned against the reference:
bit-exact on every committed reference fixture (hashes produced by the
reference's own interpret/run_compiled, tests/golden/make_golden.py) and on
the reference's known-answer tests (test_exec.cpp:26-106)."""

import json
import os

import numpy as np
import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import host as H

STREAMS = ["acceptance", "pipeline", "device"]


def _cases(stream):
    d = T.load_json(os.path.join(T.GOLDEN, f"random_{stream}.json"))
    return d["cases"]


@pytest.mark.parametrize("stream", STREAMS)
def test_oracle_matches_reference_random_graphs(stream):
    checked = 0
    for case in _cases(stream):
        ref = case["reference"]
        if "error" in ref:  # opaque library call: the reference throws too
            continue
        g = H.graph_from_json(case["bundle"]["graph"])
        inputs = T.gen_inputs(g, case["input_seed"])
        vals = T.interpret(g, inputs, mode=0)
        h = T.fnv1a([vals[o] for o in g.outputs])
        assert h == ref["interpret_fnv"], f"{stream} graph {case['bundle']['stream']['index']}"
        # the reference's block simulator agrees with its interpreter (bit-exact)
        assert ref["compiled_fnv"] == ref["interpret_fnv"]
        checked += 1
    assert checked >= 20


def test_oracle_matches_reference_configs_small():
    gold = T.load_json(os.path.join(T.GOLDEN, "configs_small.json"))
    for name, info in gold.items():
        g, rep, b = H.load_bundle(os.path.join(T.PLANS, f"{name}.small.json"))
        inputs = T.gen_inputs(g, info["seed"], info["lo"], info["hi"])
        vals = T.interpret(g, inputs, mode=0)
        assert T.fnv1a([vals[o] for o in g.outputs]) == info["reference"]["interpret_fnv"], name


def _g(instrs, outputs=None):
    if outputs is None:
        used = {o for i in instrs for o in i.get("operands", [])}
        outputs = [i["id"] for i in instrs if i["id"] not in used]
    return H.graph_from_json({"instructions": instrs, "outputs": outputs})


def test_known_answer_elementwise():  # test_exec.cpp:26-40
    g = _g([{"id": "p", "op": "parameter", "shape": [4]}, {"id": "q", "op": "parameter", "shape": [4]},
            {"id": "add", "op": "add", "operands": ["p", "q"], "shape": [4]},
            {"id": "cmp", "op": "compare", "operands": ["p", "q"], "shape": [4]},
            {"id": "sel", "op": "select", "operands": ["cmp", "p", "q"], "shape": [4]},
            {"id": "exp", "op": "exp", "operands": ["p"], "shape": [4]}])
    v = T.interpret(g, {"p": np.array([1, -2, 3, 0], np.float32), "q": np.array([4, 5, -6, 0], np.float32)})
    assert v["add"][0] == 5.0 and v["cmp"][1] == 0.0 and v["cmp"][2] == 1.0
    assert v["sel"][2] == 3.0 and v["sel"][1] == 5.0
    assert v["exp"][0] == np.float32(np.e)  # glibc expf is correctly rounded here (numpy is 1 ulp off)


def test_known_answer_reduce_fold_order():  # test_exec.cpp:42-50
    g = _g([{"id": "p", "op": "parameter", "shape": [2, 3]},
            {"id": "s", "op": "reduce", "operands": ["p"], "shape": [2], "reduce_dims": [1], "reducer": "sum"},
            {"id": "m", "op": "reduce", "operands": ["p"], "shape": [3], "reduce_dims": [0], "reducer": "max"}])
    v = T.interpret(g, {"p": np.arange(1, 7, dtype=np.float32).reshape(2, 3)})
    assert list(v["s"]) == [6.0, 15.0] and v["m"][0] == 4.0 and v["m"][2] == 6.0


def test_known_answer_shape_ops():  # test_exec.cpp:52-62
    g = _g([{"id": "p", "op": "parameter", "shape": [2, 3]},
            {"id": "t", "op": "transpose", "operands": ["p"], "shape": [3, 2], "permutation": [1, 0]},
            {"id": "r", "op": "reshape", "operands": ["p"], "shape": [6]},
            {"id": "b", "op": "broadcast", "operands": ["p"], "shape": [2, 3, 2], "broadcast_dim_map": [0, 1]}])
    v = T.interpret(g, {"p": np.arange(1, 7, dtype=np.float32).reshape(2, 3)})
    assert v["t"].ravel()[1] == 4.0 and v["r"][4] == 5.0 and v["b"].ravel()[2 * 2 + 0 * 6 + 1] == 3.0


def test_known_answer_bitcast_and_matmul():  # test_exec.cpp:64-87
    g = _g([{"id": "p", "op": "parameter", "shape": [2]},
            {"id": "b", "op": "bitcast", "operands": ["p"], "shape": [2], "dtype": "i32"},
            {"id": "u", "op": "neg", "operands": ["b"], "shape": [2], "dtype": "i32"}])
    v = T.interpret(g, {"p": np.array([1.0, -2.0], np.float32)})
    assert v["b"].view(np.float32)[0] == 1.0
    g2 = _g([{"id": "p", "op": "parameter", "shape": [1, 2, 2]}, {"id": "q", "op": "parameter", "shape": [1, 2, 2]},
             {"id": "d", "op": "batch_matmul", "operands": ["p", "q"], "shape": [1, 2, 2]}])
    v2 = T.interpret(g2, {"p": np.array([1, 2, 3, 4], np.float32).reshape(1, 2, 2),
                          "q": np.array([5, 6, 7, 8], np.float32).reshape(1, 2, 2)})
    assert v2["d"].ravel()[0] == 19.0 and v2["d"].ravel()[3] == 50.0


def test_known_answer_constants_and_missing_input():  # test_exec.cpp:94-106
    g = _g([{"id": "c", "op": "constant", "shape": [3], "value": 2.5},
            {"id": "u", "op": "neg", "operands": ["c"], "shape": [3]}])
    v = T.interpret(g, {})
    assert v["c"][2] == 2.5 and v["u"][0] == -2.5
    g2 = _g([{"id": "p", "op": "parameter", "shape": [4]}, {"id": "u", "op": "neg", "operands": ["p"], "shape": [4]}])
    with pytest.raises(RuntimeError):
        T.interpret(g2, {})


def test_generator_matches_c_restatement():
    """numpy input stream == oracle/sfx_gen.h (the stream ref_tool feeds the reference)."""
    g = _g([{"id": "a", "op": "parameter", "shape": [7, 5]}, {"id": "b", "op": "parameter", "shape": [9], "dtype": "i32"},
            {"id": "s", "op": "reduce", "operands": ["a"], "shape": [7], "reduce_dims": [1], "reducer": "sum"},
            {"id": "n", "op": "neg", "operands": ["b"], "shape": [9], "dtype": "i32"}])
    a = T.gen_tensor(7, 0, 35, "f32", -1.0, 1.0)
    assert a.min() >= -1.0 and a.max() < 1.0
    prefix = T.gen_tensor(7, 0, 10, "f32", -1.0, 1.0)
    assert np.array_equal(prefix, a[:10])
    assert np.array_equal(T.gen_tensor(7, 0, 5, "f32", -1.0, 1.0, offset=30), a[30:])
    b = T.gen_tensor(7, 1, 9, "i32")
    assert b.min() >= 1 and b.max() <= 4
    assert g.parameters()[0].id == "a"


def test_fp64_mode_is_close_to_reference_mode():
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C1.small.json"))
    inputs = T.gen_inputs(g, 42, -1.0, 1.0)
    a = T.interpret(g, inputs, 0)["y"]
    e = T.interpret(g, inputs, 1)["y"]
    assert T.strict_close(a, e)
    assert not np.array_equal(a, e)  # fp64 really differs in the low bits


@pytest.mark.skipif(not T.have_ref_tool(), reason="reference tool not built (no /root/reference here)")
def test_oracle_matches_reference_live_small_configs():
    """Live cross-check against the reference library (build container only)."""
    for name in ["C1", "C3b", "C4"]:
        path = os.path.join(T.PLANS, f"{name}.small.json")
        g, rep, b = H.load_bundle(path)
        ref = T.ref_run(path, 5, -1.0, 1.0)
        inputs = T.gen_inputs(g, 5, -1.0, 1.0)
        vals = T.interpret(g, inputs)
        got = b"".join(np.ascontiguousarray(vals[o]).tobytes() for o in g.outputs)
        assert got == ref["interpret_bytes"], name


def test_fast_generator_equals_numpy_stream():
    g, rep, b = H.load_bundle(os.path.join(T.PLANS, "C4.small.json"))
    a = T.gen_inputs(g, 3, -1.0, 1.0)
    f = T.gen_inputs_fast(g, 3, -1.0, 1.0)
    for k in a:
        assert np.array_equal(a[k], f[k])


def test_batch_slices_equal_b1_graph_on_offset_stream():
    """The C5 full-size GPU check compares batch b of the b64 output with the
    b1 graph run on batch b's slice of the input stream.  Pinned here on a
    small batch count: the oracle on the B=3 graph, sliced per batch, equals
    the oracle on the b1 graph with batch_slice_inputs — bit for bit."""
    from workloads import configs
    full = H.parse_graph(configs.c5_bert(B=3, S=32))
    small = H.parse_graph(configs.c5_bert(B=1, S=32))
    fin = T.gen_inputs_fast(full, 42, -1.0, 1.0)
    want = T.interpret(full, fin, 0)
    for b in range(3):
        sin = T.batch_slice_inputs(full, small, 42, b)
        got = T.interpret(small, sin, 0)
        for o in small.outputs:
            n = small.at(o).numel()
            assert np.array_equal(got[o].reshape(-1), want[o].reshape(-1)[b * n:(b + 1) * n]), (b, o)
