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


class HostComm:
    """Host-staged transport callbacks (ss_host_comm, ABI 5) over a torch.distributed
    group -- gloo works on any host.  Lets several processes run the distributed
    Domain on ONE GPU: each rank's halo planes and residual partials go device -> host
    -> gloo -> host -> device, with the NCCL transport's message pattern, so the
    results equal the single domain's bit for bit.  Synchronous; a test / debugging
    path, not the multi-GPU data path."""

    def __init__(self, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)

        def sendrecv(ctx, peer, send, recv, nbytes):
            try:
                s = torch.frombuffer((C.c_uint8 * nbytes).from_address(send), dtype=torch.uint8)
                r = torch.frombuffer((C.c_uint8 * nbytes).from_address(recv), dtype=torch.uint8)
                reqs = [dist.isend(s, peer, group=group), dist.irecv(r, peer, group=group)]
                for q in reqs:
                    q.wait()
                return 0
            except Exception:  # reported to the library as a transport failure
                return 1

        def allgather(ctx, local, allbuf, nbytes):
            try:
                loc = torch.frombuffer((C.c_uint8 * nbytes).from_address(local), dtype=torch.uint8)
                out = torch.frombuffer((C.c_uint8 * (nbytes * self.world)).from_address(allbuf), dtype=torch.uint8)
                dist.all_gather(list(out.chunk(self.world)), loc, group=group)
                return 0
            except Exception:
                return 1

        SR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t)
        AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)

        class _Abi(C.Structure):
            _fields_ = [("ctx", C.c_void_p), ("sendrecv", SR), ("allgather", AG)]

        self._sr, self._ag = SR(sendrecv), AG(allgather)  # kept alive with the session
        self._abi = _Abi(None, self._sr, self._ag)

    def as_abi(self):
        import ctypes as C
        return C.cast(C.pointer(self._abi), C.c_void_p)
