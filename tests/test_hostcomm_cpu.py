"""CPU: dist.HostComm -- the callbacks the host-staged transport (transport_host.cu)
calls -- in real 2- and 3-process gloo jobs: the sendrecv pattern of one colour
pass's exchange (plane 1 <-> the lower neighbour, plane n4 <-> the upper one,
lower neighbour first) and the rank-ordered all-gather of residual partials."""
import ctypes as C
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _main(rank, world, port, q):
    import torch.distributed as tdist

    from paper_2111_11866_b200 import dist as ssd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hc = ssd.HostComm()
        abi = C.cast(hc.as_abi(), C.POINTER(hc._abi.__class__)).contents
        n = 37
        planes = np.arange(4 * n, dtype=np.float64).reshape(4, n) + 1000.0 * rank  # [halo0, 1, n4, halo]
        ok = []
        if rank > 0:
            ok.append(abi.sendrecv(None, rank - 1, planes[1].ctypes.data, planes[0].ctypes.data, 8 * n))
        if rank + 1 < world:
            ok.append(abi.sendrecv(None, rank + 1, planes[2].ctypes.data, planes[3].ctypes.data, 8 * n))
        loc = np.array([rank + 0.5, rank * 2.0], dtype=np.float64)
        allv = np.zeros(2 * world)
        ok.append(abi.allgather(None, loc.ctypes.data, allv.ctypes.data, loc.nbytes))
        q.put((rank, ok, planes, allv))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hostcomm_exchange_and_allgather(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (ok, pl, av)) for r, ok, pl, av in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
    n = 37
    base = np.arange(4 * n, dtype=np.float64).reshape(4, n)
    for r in range(world):
        ok, pl, av = res[r]
        assert all(x == 0 for x in ok)
        if r > 0:  # halo 0 <- lower neighbour's plane n4 (row 2)
            assert np.array_equal(pl[0], base[2] + 1000.0 * (r - 1))
        if r + 1 < world:  # halo n4+1 <- upper neighbour's plane 1 (row 1)
            assert np.array_equal(pl[3], base[1] + 1000.0 * (r + 1))
        assert np.array_equal(av, np.array([[q + 0.5, q * 2.0] for q in range(world)]).ravel())
