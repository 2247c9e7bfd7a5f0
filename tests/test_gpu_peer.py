"""Cross-rank column combine through peer memory (opts.cross_rank), on GPU.

The batch-sharded path's one exchange is a column reduction over the batch
(C3's db).  With cross_rank=1 the column kernel itself pushes each column
tile's partial to every rank's peer arena and folds the ranks in rank order
inside the same launch (no NCCL call).  Each rank runs on its own GPU when the
box has enough of them (rank % device_count); on a 1-GPU box the ranks are
processes sharing cuda:0 through CUDA IPC — the same cuIpcOpenMemHandle path
that maps a peer GPU's arena over NVLink on a multi-GPU node.  Handles are exchanged over gloo (127.0.0.1).

Checks: every rank's db equals the fp64 restatement of the UNSHARDED graph
(rows of all ranks) within the north_star bounds and is bit-identical across
ranks; element roots (C3b's dx) stay rank-local; repeated launches and CUDA
graph replays (the per-tile sequence numbers / double-buffered slots) stay
correct with fresh inputs each time; the min fold keeps the reference's "NaN
first element wins" rule where the first element is row 0 of rank 0.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import sfx_testlib as T
from paper_1811_05213_b200 import host as H
from workloads import configs

pytestmark = pytest.mark.gpu

WS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(seed, idx, n_rows, cols, rank):
    return T.gen_tensor(seed, idx, n_rows * cols, "f32", -1.0, 1.0, offset=rank * n_rows * cols).reshape(n_rows, cols)


def _worker(rank, ws, port, case, q):
    import sys
    sys.path.insert(0, T.ROOT)
    sys.path.insert(0, os.path.join(T.ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import torch
        # distinct GPUs when the box has them (NVLink peer mapping), else both
        # ranks share cuda:0 through the same IPC path
        dev_i = rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_i)
        ctx = H.Context(dev_i)
        ctx.peer_init(rank, ws, H.torch_all_gather, nbytes=1 << 22)
        out = []
        if case in ("C3", "C3b"):
            g, rep, _ = H.load_bundle(os.path.join(T.PLANS, f"{case}.small.json"))
            n, c = g.at("dy").shape
            cg = H.CompiledGraph(ctx, g, rep, cross_rank=1)
            assert [k.info["strategy"] for k in cg.kernels][0] == "col"
            before = ctx.launch_count()
            for it in range(4):  # fresh inputs per launch: slots / sequence numbers rotate
                inputs = {"dy": _shard(100 + it, 0, n, c, rank), "x": _shard(100 + it, 1, n, c, rank)}
                res = cg.run_host(inputs)
                out.append({o: res[o] for o in g.outputs})
            assert ctx.launch_count() - before == 4 * cg.launches_per_run
            # device-resident runs with CUDA-graph replay on one buffer set
            import torch
            dev = torch.device("cuda", dev_i)
            ins = [torch.from_numpy(_shard(200, i, n, c, rank)).to(dev) for i in range(2)]
            outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
            st = torch.cuda.Stream(device=dev)
            for _ in range(3):
                cg.run([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], stream=st.cuda_stream,
                       cuda_graph=True)
            st.synchronize()
            out.append({o: t.cpu().numpy() for o, t in zip(g.outputs, outs)})
            cg.close()
        elif case == "bnsync":
            g, rep, _ = H.load_bundle(os.path.join(T.GOLDEN, "plans_extra", "bnsync_shard_2048x256.json"))
            cg = H.CompiledGraph(ctx, g, rep, cross_rank=1)
            assert [k.info["strategy"] for k in cg.kernels] == ["colbc"]
            for it in range(3):
                inputs = _bn_inputs(300 + it, rank)
                out.append(cg.run_host(inputs))
            import torch
            dev = torch.device("cuda", dev_i)
            inputs = _bn_inputs(400, rank)
            ins = [torch.from_numpy(inputs[p]).to(dev) for p in cg.param_ids]
            outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
            st = torch.cuda.Stream(device=dev)
            for _ in range(3):
                cg.run([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], stream=st.cuda_stream,
                       cuda_graph=True)
            st.synchronize()
            out.append({o: t.cpu().numpy() for o, t in zip(g.outputs, outs)})
            cg.close()
        elif case == "two_groups":
            g, rep, _ = H.load_bundle(os.path.join(T.GOLDEN, "plans_xrank", "two_xrank_shard_2048x256.json"))
            cg = H.CompiledGraph(ctx, g, rep, cross_rank=1)
            assert sorted(k.info["strategy"] for k in cg.kernels) == ["col", "colbc"]
            import torch
            dev = torch.device("cuda", dev_i)
            for it in range(2):
                inputs = _two_inputs(500 + it, rank)
                out.append(cg.run_host(inputs))
                ins = [torch.from_numpy(inputs[p]).to(dev) for p in cg.param_ids]
                outs = [torch.empty(g.at(o).shape, device=dev) for o in g.outputs]
                st = torch.cuda.Stream(device=dev)
                for _ in range(3):  # device path: the captured graph, replayed
                    cg.run([t.data_ptr() for t in ins], [t.data_ptr() for t in outs], stream=st.cuda_stream,
                           cuda_graph=True)
                st.synchronize()
                out.append({o: t.cpu().numpy() for o, t in zip(g.outputs, outs)})
            cg.close()
        elif case == "min_nan":
            g, prog, p = _min_program(rank)
            (got,) = H.run_program(prog, g, {"p": p}, ctx=ctx, cross_rank=1)
            out.append({"c2": got})
        q.put((rank, out, None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _bn_inputs(seed, rank, rows=2048, cols=256):
    """x: this rank's rows of the global batch; gamma / beta: the same on every rank."""
    return {"x": _shard(seed, 0, rows, cols, rank),
            "g": T.gen_tensor(seed, 1, cols, "f32", 0.5, 1.5),
            "b": T.gen_tensor(seed, 2, cols, "f32", -1.0, 1.0)}


def _two_inputs(seed, rank, rows=2048, cols=256):
    d = _bn_inputs(seed, rank, rows, cols)
    d["dy"] = _shard(seed, 3, rows, cols, rank)
    d["z"] = _shard(seed, 4, rows, cols, rank)
    return d


def _min_rows(rank):
    p = _shard(5, 0, 64, 128, rank).copy()
    p[0, 1::2] = np.nan     # row 0 of this shard: only rank 0's is the global first element
    p[9, ::4] = np.nan      # later NaNs: skipped
    return p


def _min_program(rank):
    doc = {"instructions": [
        {"id": "p", "op": "parameter", "shape": [64, 128]},
        {"id": "cmin", "op": "reduce", "operands": ["p"], "shape": [128], "reduce_dims": [0], "reducer": "min"},
        {"id": "c2", "op": "scale", "operands": ["cmin"], "shape": [128], "scalar": 2.0},
    ], "outputs": ["c2"]}
    g = H.graph_from_json(doc)
    prog = H.KernelProgram("c2", ["cmin", "c2"], ["c2"], 1, 64, 512,
                           [{"kind": "materialize", "instr": "cmin", "schedule": [0, 1, "row"], "dest": "shared",
                             "offset": 0, "bytes": 512}, {"kind": "barrier"},
                            {"kind": "materialize", "instr": "c2", "schedule": [0, 1, "row"], "dest": "output",
                             "root_index": 0}])
    return g, prog, _min_rows(rank)


def _spawn(case, ws=WS):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, case, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(ws)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for rank, out, err in res:
        assert err is None, f"rank {rank}: {err}"
    for p in procs:
        assert p.exitcode == 0
    return [out for _, out, _ in res]


@pytest.mark.parametrize("case,ws", [("C3", 2), ("C3b", 2), ("C3", 4)])
def test_cross_rank_column_sum(case, ws):
    g, _, _ = H.load_bundle(os.path.join(T.PLANS, f"{case}.small.json"))
    n, c = g.at("dy").shape
    outs = _spawn(case, ws)
    full = H.parse_graph(configs.c3_biasgrad(N=n * ws, C=c))
    seeds = [100, 101, 102, 103, 200]
    for i, seed in enumerate(seeds):
        dy = np.concatenate([_shard(seed, 0, n, c, r) for r in range(ws)])
        x = np.concatenate([_shard(seed, 1, n, c, r) for r in range(ws)])
        ref = T.interpret(full, {"dy": dy, "x": x}, mode=1)["db"]
        for r in range(ws):
            db = outs[r][i]["db"]
            assert T.strict_close(db, ref), (seed, r, T.mismatch_report(db, ref))
            assert np.array_equal(db.view(np.uint32), outs[0][i]["db"].view(np.uint32))  # identical on all ranks
            for o in g.outputs:  # element roots (C3b's dx_out) are rank-local
                if o != "db":
                    want = T.interpret(g, {"dy": dy[r * n:(r + 1) * n], "x": x[r * n:(r + 1) * n]}, 0)[o]
                    assert T.strict_close(outs[r][i][o], want), (o, seed, r)


def test_cross_rank_min_nan_first_rule():
    outs = _spawn("min_nan")
    g, _, _ = _min_program(0)
    full_doc = {"instructions": [
        {"id": "p", "op": "parameter", "shape": [64 * WS, 128]},
        {"id": "cmin", "op": "reduce", "operands": ["p"], "shape": [128], "reduce_dims": [0], "reducer": "min"},
        {"id": "c2", "op": "scale", "operands": ["cmin"], "shape": [128], "scalar": 2.0},
    ], "outputs": ["c2"]}
    full = H.graph_from_json(full_doc)
    p = np.concatenate([_min_rows(r) for r in range(WS)])
    want = T.interpret(full, {"p": p}, 0)["c2"]
    assert np.isnan(want[1::2]).all() and not np.isnan(want[::2]).any()
    for r in range(WS):
        got = outs[r][0]["c2"]
        assert np.array_equal(np.isnan(got), np.isnan(want)), r
        assert T.values_close(got, want), r


def test_cross_rank_sync_batchnorm():
    """SyncBatchNorm in one launch per rank: batch-norm statistics over the
    GLOBAL batch (both ranks' rows), the colbc template combining each level's
    column totals across ranks through peer memory between its grid barriers,
    then normalising this rank's rows.  Against the fp64 restatement of the
    unsharded graph; 3 host-path launches with fresh inputs + CUDA-graph replays."""
    import sys
    sys.path.insert(0, T.GOLDEN)
    from make_extra_plans import bn_graph
    outs = _spawn("bnsync")
    full = H.graph_from_json(bn_graph([2048 * WS, 256], [0], count=2048 * WS))
    for i, seed in enumerate([300, 301, 302, 400]):
        per = [_bn_inputs(seed, r) for r in range(WS)]
        inputs = {"x": np.concatenate([p["x"] for p in per]), "g": per[0]["g"], "b": per[0]["b"]}
        ref = T.interpret(full, inputs, mode=1)["y"]
        for r in range(WS):
            y = outs[r][i]["y"]
            want = ref[r * 2048:(r + 1) * 2048]
            assert T.strict_close(y, want), (seed, r, T.mismatch_report(y, want))


def test_two_cross_rank_groups_run_in_rank_order():
    """Two independent batch-crossing groups in one graph (SyncBatchNorm colbc +
    bias-grad col): both spin on peer ranks inside the kernel, so the executor
    chains them in condensation order on every rank instead of putting them on
    parallel branches (which could pair rank A's X with rank B's Y and hang).
    Host path and CUDA-graph replays, against the fp64 restatement of the
    unsharded graph."""
    import sys
    sys.path.insert(0, T.GOLDEN)
    from make_extra_plans import two_cross_rank_groups
    outs = _spawn("two_groups")
    full = H.graph_from_json(two_cross_rank_groups(rows=2048 * WS, count=2048 * WS))
    for i, seed in enumerate([500, 500, 501, 501]):
        per = [_two_inputs(seed, r) for r in range(WS)]
        inputs = {k: (np.concatenate([p[k] for p in per]) if k in ("x", "dy", "z") else per[0][k]) for k in per[0]}
        ref = T.interpret(full, inputs, mode=1)
        for r in range(WS):
            y, db = outs[r][i]["y"], outs[r][i]["db"]
            assert T.strict_close(y, ref["y"][r * 2048:(r + 1) * 2048]), (seed, r)
            assert T.strict_close(db, ref["db"]), (seed, r, T.mismatch_report(db, ref["db"]))
