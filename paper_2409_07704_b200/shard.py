"""Batch sharding across GPUs.

Items of a batch are independent -- the reference fans them out to threads
with no communication (src/parallel.cpp:130-158) -- so the multi-GPU path is
one process per GPU, each aligning a contiguous range of items.  No data
crosses NVLink and there is no collective on the data path; torch.distributed
is only used to learn rank / world size (and, optionally, to gather results).
"""

from __future__ import annotations

import numpy as np


def shard_ranges(batch: int, world: int, lengths=None):
    """Contiguous [start, stop) item ranges, one per rank.

    Without lengths the ranges differ by at most one item.  With lengths
    ([B, 2] of (t, s)) they are balanced by the work per item, t * s cells
    (the forward pass reads every valid cell once)."""
    if batch < 0 or world < 1:
        raise ValueError("batch must be >= 0 and world >= 1")
    if lengths is None:
        base, extra = divmod(batch, world)
        out, start = [], 0
        for r in range(world):
            stop = start + base + (1 if r < extra else 0)
            out.append((start, stop))
            start = stop
        return out
    lens = np.asarray(lengths, dtype=np.int64).reshape(batch, 2)
    cost = np.maximum(lens[:, 0] * lens[:, 1], 1).astype(np.float64)
    csum = np.concatenate([[0.0], np.cumsum(cost)])
    total = csum[-1]
    bounds = [0]
    for r in range(1, world):
        # first item index whose prefix cost reaches r/world of the total
        k = int(np.searchsorted(csum, total * r / world, side="left"))
        bounds.append(min(max(k, bounds[-1]), batch))
    bounds.append(batch)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _dist():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def local_range(batch: int, lengths=None, rank: int | None = None, world: int | None = None):
    """This rank's [start, stop) (rank / world from torch.distributed when
    not given)."""
    if rank is None or world is None:
        r, w = _dist()
        rank = r if rank is None else rank
        world = w if world is None else world
    return shard_ranges(batch, world, lengths)[rank]


def align_local(values, lengths=None, rank=None, world=None, **kw):
    """Aligns this rank's shard of a [B, T, S] batch.  Returns
    ((start, stop), alignment of items [start, stop))."""
    from .api import align

    B = int(values.shape[0])
    start, stop = local_range(B, lengths, rank, world)
    if stop <= start:
        return (start, stop), None
    lens = None if lengths is None else np.asarray(lengths).reshape(B, 2)[start:stop]
    return (start, stop), align(values[start:stop], lengths=lens, **kw)
