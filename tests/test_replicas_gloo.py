"""N>1 plumbing on CPU: every rank builds its own replica schedule (no data
collective), and the timing reduction is a max over ranks (gloo, world 2)."""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import paper_2312_10351_b200 as op
    from paper_2312_10351_b200 import engine, frontend, zoo
    model, x = zoo.build("googlenet")
    g = engine.static_dag(frontend.lower(model, x))
    plan = op.allocate_streams(g)
    order = op.order_opara(g, op.GPU_PRESETS["b200"]).order
    fake_seconds = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(fake_seconds, op=dist.ReduceOp.MAX)
    # bench.py: rank 0 picks the sizing variant, every replica compiles the same one
    import bench
    choice = bench.broadcast_value(dist, rank, lambda: (True, "pull", 1.5) if rank == 0 else None)
    q.put((rank, plan.num_streams, hash(order), float(fake_seconds), choice))
    dist.destroy_process_group()


def test_two_replicas_schedule_identically_and_time_is_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][1:3] == res[1][1:3] == (28, res[0][2])
    assert res[0][3] == res[1][3] == 2.0
    assert res[0][4] == res[1][4] == (True, "pull", 1.5)


class _FakeGraph:
    def __init__(self, variant, cache):
        self.bound_grids, self.splitk, self.bound_scale = variant
        self.cache = cache


def _compile_worker(rank, world, port, tmp, q):
    """bench.replica_compile's control flow with the device work stubbed: rank 0
    searches (and writes its tile choices to its own tuning cache), every other
    rank receives the variant + cache CONTENTS and builds exactly that."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import json
    from pathlib import Path

    import bench
    calls = []

    def search(cache_path):
        calls.append("search")
        Path(cache_path).write_text(json.dumps({"conv_17": [2, 64, 3]}))
        return _FakeGraph((True, "pull", 1.5), cache_path)

    def build_choice(variant, cache_path):
        calls.append("build")
        return _FakeGraph(variant, cache_path)

    rank_dir = os.path.join(tmp, f"r{rank}")   # per-rank local temp dirs (multi-node safe)
    os.makedirs(rank_dir, exist_ok=True)
    sg, variant = bench.replica_compile(dist, rank, world, search, build_choice, rank_dir)
    t = bench.time_max(dist, world, [0.5 + rank, 2.0 - rank])
    q.put((rank, calls, variant, json.loads(Path(sg.cache).read_text()), t))
    dist.destroy_process_group()


def test_replica_compile_hands_rank0_choice_to_every_rank(tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_compile_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] == ["search"] and res[1][1] == ["build"]
    assert res[0][2] == res[1][2] == (True, "pull", 1.5)
    assert res[0][3] == res[1][3] == {"conv_17": [2, 64, 3]}
    assert res[0][4] == res[1][4] == [1.5, 2.0]
