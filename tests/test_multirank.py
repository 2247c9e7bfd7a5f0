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


def test_bench_plan_per_rank():
    """Strong sharding: rank r of n runs the reference's shard plan; weak
    scaling and n = 1 run the global plan; shard counts without a plan fail."""
    import bench
    assert bench.plan_path("C5", 1).endswith("C5.full.json")
    assert bench.plan_path("C5", 8).endswith("C5.shard8.json")
    assert bench.plan_path("C5", 8, "weak").endswith("C5.full.json")
    with pytest.raises(SystemExit):
        bench.plan_path("C5", 3)
    c = bench.config_obj("C5", 8)
    assert c["shard"] == {"dim": "B", "ranks": 8, "per_rank": {"B": 8, "S": 512}, "global": {"B": 64, "S": 512}}
    assert "column kernel" in bench.config_obj("C3", 4)["parallelism"]


def test_bench_gpus_mismatch_and_self_launch():
    """--gpus N must agree with WORLD_SIZE; without torchrun, --gpus N
    re-launches bench.py as N ranks (here the CPU reference arm: rank 0 prints
    the line with n_gpus = N, the other ranks exit 0)."""
    import json
    import subprocess
    import sys
    bench = os.path.join(T.ROOT, "bench.py")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, bench, "--gpus", "2", "--impl", "reference", "--config", "C1"],
                       env=dict(env, WORLD_SIZE="1"), capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
    r = subprocess.run([sys.executable, bench, "--gpus", "2", "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "3"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert lines[0]["config"]["shard"]["per_rank"] == {"R": 4096, "C": 1024}
