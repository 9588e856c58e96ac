"""Multi-GPU host logic on CPU: batch shards, exercised with
world-size-2 gloo process groups."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_07704_b200.shard import local_range, shard_ranges


def test_even_ranges_cover_once():
    for B in (0, 1, 7, 32, 256):
        for world in (1, 2, 3, 4, 8):
            rs = shard_ranges(B, world)
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_weighted_ranges_balance_cells():
    rng = np.random.default_rng(0)
    t = rng.integers(100, 201, 256)
    s = np.minimum(800, 3 * t + rng.integers(0, 101, 256))
    lens = np.stack([t, s], 1)
    for world in (2, 4, 8):
        rs = shard_ranges(256, world, lens)
        assert rs[0][0] == 0 and rs[-1][1] == 256
        cost = [int((lens[a:b, 0] * lens[a:b, 1]).sum()) for a, b in rs]
        assert max(cost) <= (sum(cost) / world) * 1.1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, stop = local_range(B)
        # every rank reports its range; rank 0 checks the cover
        got = [None] * world
        dist.all_gather_object(got, (rank, start, stop))
        # the bench's per-rank input shard: items [r*32, r*32+32) of a
        # 32*world batch -- weak scaling, no data-path collective
        t = torch.tensor([float(stop - start)])
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        if rank == 0:
            q.put((got, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_ranges():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 33, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, total = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = sorted(got)
    assert got == [(0, 0, 17), (1, 17, 33)]
    assert total == 33.0
