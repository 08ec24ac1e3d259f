"""CPU model of the NVLink halo-push protocol (SSB_P2P).

Each "rank" is a thread owning a 1D slab of a red-black relaxation with the GPU
path's buffer discipline: iteration n reads state in(n) and writes out(n)
(out(n) = 1 + (n-1) % 3, in(1) = guess), a pass writes its own colour and pushes
its first / last owned cell into the neighbours' halo cells of the same buffer,
and passes are ordered only by per-pass counters: before pass k a rank waits
until both neighbours have signalled k-1, after it it signals k.  Random delays
shake the interleavings; the result must equal the single-domain sweep bit for
bit (any missing wait or buffer reuse race would read a stale or a future halo).
"""
import random
import threading
import time

import numpy as np
import pytest

N_CELLS, W_RANKS, ITERS, OMEGA = 37, 4, 12, 1.3


def out_buf(n):
    return 1 + (n - 1) % 3


def in_buf(n):
    return 0 if n == 1 else out_buf(n - 1)


def relax(u_in, u_out, colour, lo, hi, rhs):
    """red (colour 0) reads its neighbours from u_in, black from u_out (this iteration's
    red values); updates the cells of `colour` in [lo, hi) into u_out."""
    src = u_in if colour == 0 else u_out
    for i in range(lo, hi):
        if (i & 1) != colour:
            continue
        ubar = 0.5 * (src[i - 1] + src[i + 1]) + rhs[i]
        u_out[i] = OMEGA * ubar + (1.0 - OMEGA) * u_in[i]


def reference(u0, rhs):
    B = [u0.copy() for _ in range(4)]
    for n in range(1, ITERS + 1):
        for c in (0, 1):
            relax(B[in_buf(n)], B[out_buf(n)], c, 1, N_CELLS + 1, rhs)
    return B[out_buf(ITERS)]


@pytest.mark.parametrize("seed", range(4))
def test_push_protocol_matches_single_domain(seed):
    rng = np.random.default_rng(seed)
    u0 = np.zeros(N_CELLS + 2)
    u0[1:-1] = rng.random(N_CELLS)
    rhs = 0.01 * rng.random(N_CELLS + 2)
    want = reference(u0, rhs)

    chunk = -(-N_CELLS // W_RANKS)
    ranges = [(1 + r * chunk, min(N_CELLS, (r + 1) * chunk)) for r in range(W_RANKS)]
    # per rank: 4 buffers over the GLOBAL index space (only owned cells + 2 halos are used)
    bufs = [[u0.copy() for _ in range(4)] for _ in range(W_RANKS)]
    counters = [[0, 0] for _ in range(W_RANKS)]  # [written by low neighbour, by high neighbour]
    lock = threading.Condition()
    delays = random.Random(seed)

    def wait(r, k):
        with lock:
            lock.wait_for(lambda: (r == 0 or counters[r][0] >= k) and (r == W_RANKS - 1 or counters[r][1] >= k))

    def signal(r, k):
        with lock:
            if r > 0:
                counters[r - 1][1] = k
            if r < W_RANKS - 1:
                counters[r + 1][0] = k
            lock.notify_all()

    def rank(r):
        lo, hi = ranges[r]
        k = 0
        for n in range(1, ITERS + 1):
            for c in (0, 1):
                k += 1
                wait(r, k - 1)
                time.sleep(delays.random() * 1e-4)
                B = bufs[r]
                relax(B[in_buf(n)], B[out_buf(n)], c, lo, hi + 1, rhs)
                # push the boundary cells of this colour into the neighbours' halos
                for cell, nb in ((lo, r - 1), (hi, r + 1)):
                    if 0 <= nb < W_RANKS and (cell & 1) == c:
                        bufs[nb][out_buf(n)][cell] = B[out_buf(n)][cell]
                signal(r, k)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(W_RANKS)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    got = np.zeros(N_CELLS + 2)
    for r, (lo, hi) in enumerate(ranges):
        got[lo:hi + 1] = bufs[r][out_buf(ITERS)][lo:hi + 1]
    assert np.array_equal(got[1:-1], want[1:-1])
