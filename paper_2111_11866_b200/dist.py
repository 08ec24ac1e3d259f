"""Multi-GPU host side: the t-slab partition (Partition::create, parallel.cpp:9-19),
slab views of host arrays and the NCCL bootstrap over torch.distributed.

One process per GPU.  Rank r owns global slices ``l_begin .. l_begin+count-1``
(1-based); its host arrays are the padded planes ``l_begin-1 .. l_begin+count``
of the global padded array (owned planes plus one halo/ghost plane each side).
"""
from __future__ import annotations

import numpy as np


def partition(n4: int, world: int):
    """[(l_begin, count)] per rank; chunk ceil(n4/world), the last takes the remainder."""
    if n4 < 1 or world < 1:
        raise ValueError("n4 and world must be >= 1")
    chunk = (n4 + world - 1) // world
    last = n4 - (world - 1) * chunk
    if last < 1:
        raise ValueError(f"Partition: {world} workers leave the last one with {last} slices of {n4}")
    return [(r * chunk + 1, chunk if r < world - 1 else last) for r in range(world)]


def clamp_workers(n4: int, requested: int) -> int:
    """parallel.cpp:21-27"""
    for w in range(min(requested, n4), 1, -1):
        if n4 - (w - 1) * ((n4 + w - 1) // w) >= 1:
            return w
    return 1


def slab_view(global_padded: np.ndarray, l_begin: int, count: int) -> np.ndarray:
    """Padded planes l_begin-1 .. l_begin+count of a (n4+2, ...) array (a view)."""
    return global_padded[l_begin - 1: l_begin + count + 1]


def owned_planes(slab_padded: np.ndarray) -> np.ndarray:
    return slab_padded[1:-1]


def broadcast_uid(uid: bytes | None, group=None) -> bytes:
    """Share rank 0's NCCL unique id with every rank (any torch.distributed backend)."""
    import torch
    import torch.distributed as dist
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def reduce_slice_partials(partials_by_rank):
    """The stopping-test sum: per-slice partials of every rank, concatenated in rank
    (= global l) order and summed sequentially -- what every rank computes after
    the all-gather, so the decision is identical everywhere and independent of
    the number of ranks (solver.cpp:195-199)."""
    total = 0.0
    for part in partials_by_rank:
        for v in part:
            total += float(v)
    return total
