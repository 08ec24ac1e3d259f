"""Multi-process (world_size 2 and 3, gloo on CPU) checks of the t-slab protocol the
NCCL path implements:

* Partition semantics (parallel.cpp:9-19) and slab views of host arrays;
* the NCCL unique-id bootstrap helper (broadcast over torch.distributed);
* a numpy restatement of the slab-decomposed red-black SOR -- owned planes plus
  one halo plane per side, global colour parity, the just-updated colour's
  boundary planes exchanged after every pass (gloo send/recv), per-slice
  residuals all-gathered and summed in global l order -- which must reproduce
  the single-domain oracle bit for bit at every world size.

Test infrastructure: the GPU code path itself is checked by tests/test_gpu_slabs.py
(same protocol, device-copy transport) on one GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import _cases as cs

from paper_2111_11866_b200 import dist as ssd


def test_partition_semantics():
    assert ssd.partition(10, 3) == [(1, 4), (5, 4), (9, 2)]
    assert ssd.partition(64, 8) == [(1 + 8 * r, 8) for r in range(8)]
    with pytest.raises(ValueError):
        ssd.partition(6, 4)  # chunk 2 leaves the last worker 0 slices
    assert ssd.clamp_workers(6, 4) == 3
    assert ssd.clamp_workers(6, 5) == 3
    assert ssd.clamp_workers(7, 3) == 3
    a = np.arange(12 * 2).reshape(12, 2)
    v = ssd.slab_view(a, 5, 4)
    assert v.shape == (6, 2) and v[0, 0] == a[4, 0] and v[-1, 0] == a[9, 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sweep(u, c, rhs, omega, colour, l_glob0):
    """One colour half-sweep on a padded slab (solver.cpp:292-313), vectorised; returns
    per-slice sums of res^2 (black) -- elementwise IEEE ops in the reference's order."""
    L4, K, J, I = u.shape
    l = np.arange(L4)[:, None, None, None] + l_glob0
    k = np.arange(K)[None, :, None, None]
    j = np.arange(J)[None, None, :, None]
    i = np.arange(I)[None, None, None, :]
    sel = ((i + j + k + l) & 1) == colour
    inner = np.zeros(u.shape, bool)
    inner[1:-1, 1:-1, 1:-1, 1:-1] = True
    m = sel & inner
    cf = [c[..., f] for f in range(8)]
    nb = [np.roll(u, 1, 3), np.roll(u, -1, 3), np.roll(u, 1, 2), np.roll(u, -1, 2),
          np.roll(u, 1, 1), np.roll(u, -1, 1), np.roll(u, 1, 0), np.roll(u, -1, 0)]
    dg = 1.0 - (cf[0] + cf[1] + cf[2] + cf[3] + cf[4] + cf[5] + cf[6] + cf[7])
    acc = rhs.copy()
    for f in range(8):
        acc = acc - cf[f] * nb[f]
    ubar = acc / dg
    unew = omega * ubar + (1.0 - omega) * u
    res = dg * (unew - ubar)
    u[m] = unew[m]
    return np.where(m, res * res, 0.0)


def _red_res(u, c, rhs, l_glob0):
    L4, K, J, I = u.shape
    l = np.arange(L4)[:, None, None, None] + l_glob0
    k = np.arange(K)[None, :, None, None]
    j = np.arange(J)[None, None, :, None]
    i = np.arange(I)[None, None, None, :]
    m = (((i + j + k + l) & 1) == 0)
    inner = np.zeros(u.shape, bool)
    inner[1:-1, 1:-1, 1:-1, 1:-1] = True
    m &= inner
    cf = [c[..., f] for f in range(8)]
    nb = [np.roll(u, 1, 3), np.roll(u, -1, 3), np.roll(u, 1, 2), np.roll(u, -1, 2),
          np.roll(u, 1, 1), np.roll(u, -1, 1), np.roll(u, 1, 0), np.roll(u, -1, 0)]
    dg = 1.0 - (cf[0] + cf[1] + cf[2] + cf[3] + cf[4] + cf[5] + cf[6] + cf[7])
    res = dg * u - rhs
    for f in range(8):
        res = res + cf[f] * nb[f]
    return np.where(m, res * res, 0.0)


def _exchange(u, rank, world):
    """Boundary planes to the l-neighbours' halos (gloo send/recv; the NCCL transport
    sends only the just-updated colour, this restatement sends the whole plane)."""
    if rank > 0:
        dist.send(torch.from_numpy(np.ascontiguousarray(u[1])), rank - 1)
        buf = torch.empty(u[0].shape, dtype=torch.float64)
        dist.recv(buf, rank - 1)
        u[0] = buf.numpy()
    if rank + 1 < world:
        buf = torch.empty(u[-1].shape, dtype=torch.float64)
        dist.recv(buf, rank + 1)
        u[-1] = buf.numpy()
        dist.send(torch.from_numpy(np.ascontiguousarray(u[-2])), rank + 1)


def _worker(rank, world, port, dims, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_py as op
        g = op.Grid.make(dims, 0.25)
        u_full = cs.rand_field(dims, 3)
        st, off, _, _ = op.oracle().assemble_step(g, u_full, cs.rand_G(dims, 4), 0.6, 1e-3)
        c_full = off.astype(np.float32).astype(np.float64)  # the packed fp32 rows
        rhs_full = cs.rand_field(dims, 5)
        uid = ssd.broadcast_uid(b"x" * 128 if rank == 0 else None)
        assert uid == b"x" * 128
        lb, cnt = ssd.partition(dims[3], world)[rank]
        u = ssd.slab_view(u_full, lb, cnt).copy()
        c = ssd.slab_view(c_full, lb, cnt)
        rhs = ssd.slab_view(rhs_full, lb, cnt)
        chunk = ssd.partition(dims[3], world)[0][1]
        it = 0
        while True:
            _sweep(u, c, rhs, 1.4, 0, lb - 1)
            _exchange(u, rank, world)
            bsq = _sweep(u, c, rhs, 1.4, 1, lb - 1)
            _exchange(u, rank, world)
            rsq = _red_res(u, c, rhs, lb - 1)
            slices = np.zeros(chunk)
            for ll in range(1, cnt + 1):  # per-slice: black + red (solver.cpp:359)
                slices[ll - 1] = bsq[ll].sum() + rsq[ll].sum()
            gathered = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(slices))
            parts = [gt.numpy()[: ssd.partition(dims[3], world)[r][1]] for r, gt in enumerate(gathered)]
            res = np.sqrt(ssd.reduce_slice_partials(parts))
            it += 1
            if res <= 1e-11 or it >= 500:
                break
        q.put((rank, lb, cnt, it, u[1:-1].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_matches_oracle(oracle, world):
    dims = (5, 4, 3, 7)
    g = cs.grid(dims, 0.25)
    u_full = cs.rand_field(dims, 3)
    st, off, _, _ = oracle.assemble_step(g, u_full, cs.rand_G(dims, 4), 0.6, 1e-3)
    rhs_full = cs.rand_field(dims, 5)
    st, uo, ito, reso = oracle.redblack_sor(g, off, rhs_full, u_full, 1.4, 1e-11, 500)
    assert st == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lb, cnt, it, owned in outs:
        assert it == ito
        ref = uo[lb: lb + cnt]
        # the vectorised sweep is the same IEEE operation sequence per doxel
        assert np.array_equal(owned[:, 1:-1, 1:-1, 1:-1].view(np.uint64),
                              ref[:, 1:-1, 1:-1, 1:-1].view(np.uint64))
