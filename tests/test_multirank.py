"""N>1 host logic on CPU (gloo, world_size 2, 127.0.0.1).

The path shards by batch: every rank runs its own instance, and the only
exchange is the column sum of a batch-crossing reduction (C3's db), combined
with an all-reduce — on GPUs by sfx_allreduce_sum_f32 (NCCL), here by gloo
with the oracle standing in for the kernel.  Also checks the benchmark's
max-over-ranks timing reduction.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import sfx_testlib as T
from paper_1811_05213_b200 import host as H
from workloads import configs

N, C, SEED = 256, 64, 11


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    import sys
    sys.path.insert(0, T.ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    g = H.parse_graph(configs.c3_biasgrad(N=N, C=C))
    # this rank's batch shard = rows [rank*N, (rank+1)*N) of the global stream
    dy = T.gen_tensor(SEED, 0, N * C, "f32", -1.0, 1.0, offset=rank * N * C).reshape(N, C)
    x = T.gen_tensor(SEED, 1, N * C, "f32", -1.0, 1.0, offset=rank * N * C).reshape(N, C)
    part = T.interpret(g, {"dy": dy, "x": x}, mode=1)["db"]
    t = torch.from_numpy(part.astype(np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    q.put((rank, t.numpy().astype(np.float32), float(ms.item())))
    dist.destroy_process_group()


def test_batch_sharded_column_sum_two_ranks():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = H.parse_graph(configs.c3_biasgrad(N=N * ws, C=C))
    inputs = T.gen_inputs(full, SEED, -1.0, 1.0)
    ref = T.interpret(full, inputs, mode=1)["db"]
    for rank, db, ms in res:
        assert T.strict_close(db, ref), T.mismatch_report(db, ref)
        assert ms == float(ws)  # max over ranks


def test_bench_rank_environment_defaults(monkeypatch):
    import bench
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_env() == (1, 0, 0)
    monkeypatch.setenv("WORLD_SIZE", "8")
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("LOCAL_RANK", "3")
    assert bench.dist_env() == (8, 3, 3)


def _rounds_worker(rank, ws, port, q):
    import sys
    sys.path.insert(0, T.ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    local_want = 3 if rank == 0 else 7  # the ranks' own stopping points differ
    done = []
    n = bench.agreed_rounds(lambda: len(done) < local_want, lambda: done.append(1), ws, "cpu")
    q.put((rank, n, len(done)))
    dist.destroy_process_group()


def test_bench_load_rounds_agree_across_ranks():
    """bench.py's clock-sampling load phases stop on local timing; with a
    cross-rank step the ranks must still run the same number of rounds."""
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rounds_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [7, 7] and [r[2] for r in res] == [7, 7]
