"""The t-slab decomposition on one GPU: a grid split into n slabs
that exchange halo planes and all-gather per-slice residuals must give the
single-slab result bit for bit (same iterates, same iteration counts) -- the
property the multi-GPU NCCL path relies on."""
import os
import sys

import numpy as np
import pytest

import _cases as cs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def run(ss, g, image, rows, params, n_slabs, steps, u0=None, mode=0):
    with ss.Session(g, n_slabs=n_slabs) as s:
        s.set_loop_mode(mode)
        s.prepare(image, rows, params, u0)
        diags = [s.step() for _ in range(steps)]
        return s.get_u(), [d["iterations"] for d in diags], diags, s.get_mask(0.5)


@pytest.mark.parametrize("n_slabs", [2, 3, 6])
def test_slabs_match_single_golden(gpu, n_slabs):
    d = dict(np.load(os.path.join(GOLD, "segment.npz")))
    dims = tuple(int(x) for x in d["dims"])
    h = float(d["h"])
    g = gpu.Grid.make(dims, h)
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=3, sigma=np.sqrt(2) * h, K=200.0,
                       delta=0.5, vartheta=0.5, rescale_radius=3.0, sor_rel_tol=1e-8)
    u, its, diags, mask = run(gpu, g, d["image"], d["rows"], p, n_slabs, 3)
    assert its == list(d["iters_rel"])
    assert np.array_equal(u.view(np.uint64), d["u_rel"].view(np.uint64))
    assert np.array_equal(mask, (d["u_rel"][g.interior] >= 0.5).astype(np.uint8))
    np.testing.assert_allclose([x["tol"] for x in diags], d["tol_rel"], rtol=1e-13)


@pytest.mark.parametrize("dims,n_slabs", [((9, 7, 6, 7), 3), ((10, 8, 5, 9), 2), ((8, 6, 6, 5), 5)])
def test_slabs_odd_offsets(gpu, oracle, dims, n_slabs):
    """Slab offsets with odd l0 exercise the global colour parity; compared with the oracle."""
    from oracle import oracle_py as op
    h = 1.0 / dims[0]
    g = gpu.Grid.make(dims, h)
    img = cs.f32_image(dims, 5)
    rows = [(f, (dims[0] - 1) / 2, (dims[1] - 1) / 2, (dims[2] - 1) / 2, 1.5) for f in range(dims[3])]
    rows += [(dims[3] // 2, 1.0, 1.0, 1.0, 2.0)]
    kw = dict(tau=h, epsilon=1e-3, omega=1.4, n_steps=2, sigma=np.sqrt(2) * h, K=300.0, delta=0.5,
              vartheta=0.5, rescale_radius=3.0, sor_rel_tol=1e-8, smooth_steps=2)
    u, its, _, _ = run(gpu, g, img, rows, gpu.seg_params(**kw), n_slabs, 2)
    st, uo, info = op.oracle().segment(op.Grid.make(dims, h), img, rows, op.seg_params(**kw))
    assert st == 0
    assert its == [x["iterations"] for x in info["diags"]]
    assert np.array_equal(u.view(np.uint64), uo.view(np.uint64))


def test_slabs_fixed_sweeps(gpu):
    dims = (12, 10, 8, 8)
    h = 1.0 / 12
    g = gpu.Grid.make(dims, h)
    img = cs.f32_image(dims, 9)
    rows = [(f, 5.5, 4.5, 3.5, 1.5) for f in range(dims[3])]
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=1, sigma=np.sqrt(2) * h, K=100.0,
                       delta=0.5, vartheta=0.5, rescale_radius=3.0)
    outs = []
    for n in (1, 4):
        with gpu.Session(g, n_slabs=n) as s:
            s.prepare(img, rows, p)
            r = s.fixed_sweeps(20)
            outs.append((r, s.get_u()))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1].view(np.uint64), outs[1][1].view(np.uint64))


def test_nccl_session_world1(gpu):
    """The NCCL transport end to end at world size 1 (dlopen, comm init, all-gather
    of slice residuals, slab-shaped host arrays): identical to the plain session."""
    d = dict(np.load(os.path.join(GOLD, "segment.npz")))
    dims = tuple(int(x) for x in d["dims"])
    h = float(d["h"])
    g = gpu.Grid.make(dims, h)
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=3, sigma=np.sqrt(2) * h, K=200.0,
                       delta=0.5, vartheta=0.5, rescale_radius=3.0, sor_rel_tol=1e-8)
    uid = gpu.nccl_unique_id()
    with gpu.Session(g, dist=(0, 1, uid)) as s:
        assert s.distributed and s.host_shape == g.shape and s.l_begin == 1 and s.l_count == dims[3]
        s.prepare(d["image"], d["rows"], p)
        its = [s.step()["iterations"] for _ in range(3)]
        u = s.get_u()
    assert its == list(d["iters_rel"])
    assert np.array_equal(u.view(np.uint64), d["u_rel"].view(np.uint64))


@pytest.mark.parametrize("kernel", ["ldg", "tma", "wave", "resident", "auto", "tma2d", "kwave"])
def test_pass_kernels_agree(gpu, kernel):
    """Both SOR colour-pass kernels give the golden segment() result bit for bit."""
    d = dict(np.load(os.path.join(GOLD, "segment.npz")))
    dims = tuple(int(x) for x in d["dims"])
    h = float(d["h"])
    g = gpu.Grid.make(dims, h)
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=3, sigma=np.sqrt(2) * h, K=200.0,
                       delta=0.5, vartheta=0.5, rescale_radius=3.0, sor_rel_tol=1e-8)
    for n_slabs in (1, 3):
        with gpu.Session(g, n_slabs=n_slabs) as s:
            s.set_kernel(kernel)
            s.prepare(d["image"], d["rows"], p)
            its = [s.step()["iterations"] for _ in range(3)]
            u = s.get_u()
        assert its == list(d["iters_rel"])
        assert np.array_equal(u.view(np.uint64), d["u_rel"].view(np.uint64))


@pytest.mark.parametrize("dims", [(7, 5, 6, 4), (33, 9, 5, 3), (130, 6, 9, 2), (1, 3, 2, 5)])
def test_kernels_agree_odd_shapes(gpu, oracle, dims):
    """Every SOR kernel (TMA two-pass, LDG two-pass, resident single launch) against the
    oracle's segment() on odd shapes: identical iterates and iteration counts."""
    h = 1.0 / max(dims[:3])
    g = gpu.Grid.make(dims, h)
    img = cs.f32_image(dims, sum(dims), noise=0.05)
    rows = [(f, (dims[0] - 1) / 2, (dims[1] - 1) / 2, (dims[2] - 1) / 2, 1.5) for f in range(dims[3])]
    kw = dict(tau=h, epsilon=1e-3, omega=1.4, sor_rel_tol=1e-8, n_steps=2, sigma=np.sqrt(2) * h, K=100.0,
              delta=0.5, vartheta=0.5, rescale_radius=2.0)
    st, uo, info = oracle.segment(cs.grid(dims, h), img, rows, oracle_params(kw))
    assert st == 0
    for kernel in ("tma", "ldg", "resident", "tma2d", "kwave"):
        with gpu.Session(g) as s:
            s.set_kernel(kernel)
            s.prepare(img, rows, gpu.seg_params(**kw))
            its = [s.step()["iterations"] for _ in range(2)]
            u = s.get_u()
        assert its == [x["iterations"] for x in info["diags"]], kernel
        assert np.array_equal(u.view(np.uint64), uo.view(np.uint64)), kernel


def oracle_params(kw):
    from oracle.oracle_py import seg_params
    return seg_params(**kw)


def test_halo_exchange_timing(gpu):
    """Profiling mode times the halo exchanges of a multi-slab solve (comm stream) and the
    part the compute stream waited for (bench.py's "halo" object for N > 1): every
    exchange of the timed passes is counted, and results are unchanged by the timing."""
    dims = (12, 10, 8, 8)
    h = 1.0 / 12
    g = gpu.Grid.make(dims, h)
    img = cs.f32_image(dims, 9)
    rows = [(f, 5.5, 4.5, 3.5, 1.5) for f in range(dims[3])]
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=1, sigma=np.sqrt(2) * h, K=100.0,
                       delta=0.5, vartheta=0.5, rescale_radius=3.0)
    outs = []
    for prof in (False, True):
        with gpu.Session(g, n_slabs=4) as s:
            s.set_kernel("ldg")  # exchange copies between the passes (no in-kernel halo push)
            s.prepare(img, rows, p)
            s.set_profiling(prof)
            s.profile()
            r = s.fixed_sweeps(12)
            pr = s.profile()
            outs.append((r, s.get_u()))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1].view(np.uint64), outs[1][1].view(np.uint64))
    assert pr["halo_n"] == pr["red_n"] + pr["black_n"] >= 2 * 12  # one exchange per colour pass
    assert pr["halo_ms"] > 0.0
    assert 0.0 <= pr["halo_exposed_ms"] <= pr["red_ms"] + pr["black_ms"]


@pytest.mark.parametrize("dims", [(64, 16, 12, 10), (32, 24, 9, 7), (40, 8, 5, 13), (1, 3, 2, 5)])
def test_kwave_matches_two_pass(gpu, dims):
    """The one-sweep k-wavefront kernel (red and black items of one iteration in one
    launch, black items waiting on per-item flags of the red items they read) gives the
    two-pass TMA kernel's iterates bit for bit, with the same iteration counts."""
    h = 1.0 / max(dims[:3])
    g = gpu.Grid.make(dims, h)
    img = cs.f32_image(dims, 3 + sum(dims), noise=0.05)
    rows = [(f, (dims[0] - 1) / 2, (dims[1] - 1) / 2, (dims[2] - 1) / 2, 2.5) for f in range(dims[3])]
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, sor_rel_tol=1e-8, n_steps=3, sigma=np.sqrt(2) * h,
                       K=100.0, delta=0.5, vartheta=0.5, rescale_radius=3.0)
    out = {}
    for kernel in ("tma", "kwave"):
        for mode in (0, 1):  # host-driven loop / CUDA-graph conditional loop
            with gpu.Session(g) as s:
                s.set_kernel(kernel)
                s.set_loop_mode(mode)
                s.prepare(img, rows, p)
                its = [s.step()["iterations"] for _ in range(3)]
                assert s.sor_kernel() == kernel
                out[kernel, mode] = (its, s.get_u())
    ref_its, ref_u = out["tma", 1]
    for key, (its, u) in out.items():
        assert its == ref_its, key
        assert np.array_equal(u.view(np.uint64), ref_u.view(np.uint64)), key


_NOPUSH_SCRIPT = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, os.environ["REPO"])
import paper_2111_11866_b200 as ss
d = dict(np.load(os.path.join(os.environ["REPO"], "tests", "golden", "segment.npz")))
dims = tuple(int(x) for x in d["dims"])
h = float(d["h"])
g = ss.Grid.make(dims, h)
p = ss.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=3, sigma=np.sqrt(2) * h, K=200.0,
                  delta=0.5, vartheta=0.5, rescale_radius=3.0, sor_rel_tol=1e-8)
out = {}
for n_slabs in (2, 3):
    with ss.Session(g, n_slabs=n_slabs) as s:
        s.set_kernel(os.environ["KERNEL"])
        s.prepare(d["image"], d["rows"], p)
        s.set_profiling(True)  # counts the exchanges: proves the exchange (not push) path ran
        s.profile()
        its = [s.step()["iterations"] for _ in range(3)]
        halo_n = s.profile()["halo_n"]
        u = s.get_u()
    out[n_slabs] = (its == list(d["iters_rel"]),
                    bool(np.array_equal(u.view(np.uint64), d["u_rel"].view(np.uint64))), halo_n,
                    list(dims))
print(json.dumps({str(k): v for k, v in out.items()}))
"""


@pytest.mark.parametrize("kernel", ["tma", "tma2d"])
def test_slabs_exchange_path_tma(gpu, kernel):
    """Slab groups WITHOUT the in-kernel halo push (SSB_PUSH=0, the path NCCL ranks take):
    the two end slices in one strided TMA launch on the high-priority stream, the interior
    with dynamic items on the main stream, exchange copies on the comm stream, the decision
    on its own stream overlapped with the black pass -- bit-identical to the golden
    single-domain run.  (SSB_PUSH is read once per process: a subprocess.)"""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SSB_PUSH="0", REPO=repo, KERNEL=kernel)
    r = subprocess.run([sys.executable, "-c", _NOPUSH_SCRIPT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for k, (its_ok, u_ok, halo_n, dims) in res.items():
        assert its_ok and u_ok, (kernel, k, res)
        assert halo_n > 0, (kernel, k, res)


@pytest.mark.parametrize("n_slabs,pinned", [(1, True), (1, False), (3, False)])
def test_step_host_matches_device_steps(gpu, n_slabs, pinned):
    """ss_session_step_host (compact host interiors in and out; single slab + page-locked
    input: chunked upload overlapped with the per-chunk assembly) == set_u + step + get_u."""
    import torch
    import workloads
    wl = workloads.small((20, 14, 10, 11), seed=21)
    g = gpu.Grid.make(wl.dims, wl.h)
    p = gpu.seg_params(**{**wl.params, "n_steps": 6, "sor_rel_tol": 1e-8, "rescale_radius": 3.0})
    inner = (slice(1, -1),) * 4
    with gpu.Session(g, n_slabs=n_slabs) as a, gpu.Session(g) as b:
        a.prepare(wl.image, wl.rows, p, wl.u0)
        b.prepare(wl.image, wl.rows, p, wl.u0)
        shape = a.interior_shape
        if pinned:
            t_in = torch.empty(shape, dtype=torch.float64).pin_memory()
            t_out = torch.empty(shape, dtype=torch.float64).pin_memory()
            t_in.copy_(torch.from_numpy(np.ascontiguousarray(b.get_u()[inner])))
        else:
            h_in = np.ascontiguousarray(b.get_u()[inner])
            h_out = np.empty(shape)
        for n, fixed in enumerate([0, 0, 9, 0]):
            if pinned:
                da = a.step_host(t_in.data_ptr(), t_out.data_ptr(), fixed)
                got = t_out.numpy().copy()
                t_in, t_out = t_out, t_in
            else:
                da = a.step_host(h_in, h_out, fixed)
                got = h_out.copy()
                h_in, h_out = h_out, h_in
            db = b.step_fixed(fixed) if fixed else b.step()
            want = b.get_u()[inner]
            # the single-slab session runs the resident kernel on this small grid, the slab
            # group the TMA two-pass: same iterates, residual sums in a different order
            assert [da[k] for k in ("iterations", "umin", "umax")] == [db[k] for k in ("iterations", "umin", "umax")], n
            assert da["residual"] == pytest.approx(db["residual"], rel=1e-12) and da["tol"] == db["tol"], n
            assert np.array_equal(got.view(np.uint64), np.ascontiguousarray(want).view(np.uint64)), n
        # the interior copies alone
        a.set_u_interior(want * 0.5)
        assert np.array_equal(a.get_u_interior(), want * 0.5)


@pytest.mark.parametrize("chunks_slices", [(20, 14, 10, 11), (16, 12, 8, 5)])
def test_step_host_async_chain_matches_device_steps(gpu, chunks_slices):
    """ss_session_step_host_async (ABI 6): the result's download left in flight, the next
    step's upload of that same buffer chained to it on the device chunk by chunk -- K steps
    through host memory == K device steps bit for bit, with a mid-run switch to a fresh input
    buffer (not chained: waits for the download first) and the synchronous call in between."""
    import torch
    import workloads
    wl = workloads.small(chunks_slices, seed=23)
    g = gpu.Grid.make(wl.dims, wl.h)
    p = gpu.seg_params(**{**wl.params, "n_steps": 8, "sor_rel_tol": 1e-8, "rescale_radius": 3.0})
    inner = (slice(1, -1),) * 4
    with gpu.Session(g) as a, gpu.Session(g) as b:
        a.prepare(wl.image, wl.rows, p, wl.u0)
        b.prepare(wl.image, wl.rows, p, wl.u0)
        shape = a.interior_shape
        bufs = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in range(3)]
        bufs[0].copy_(torch.from_numpy(np.ascontiguousarray(b.get_u()[inner])))
        order = [(0, 1, 0), (1, 0, 0), (0, 1, 7), (2, 0, 0), (0, 1, 0), (1, 2, 5)]
        for n, (i, o, fixed) in enumerate(order):
            if i == 2:  # a fresh input buffer: the host copies the last result into it
                a.wait()
                bufs[2].copy_(bufs[1 if order[n - 1][1] == 1 else 0])
            if n == 3:
                da = a.step_host(bufs[i].data_ptr(), bufs[o].data_ptr(), fixed)
            else:
                da = a.step_host_async(bufs[i].data_ptr(), bufs[o].data_ptr(), fixed)
            db = b.step_fixed(fixed) if fixed else b.step()
            assert [da[k] for k in ("iterations", "umin", "umax")] == [db[k] for k in ("iterations", "umin", "umax")], n
            a.wait()
            want = np.ascontiguousarray(b.get_u()[inner])
            assert np.array_equal(bufs[o].numpy().view(np.uint64), want.view(np.uint64)), n
        # a chain of async steps with every input still on its way down, waited for once
        a.wait()
        bufs[0].copy_(torch.from_numpy(np.ascontiguousarray(b.get_u()[inner])))
        for n in range(5):
            fixed = 6 if n == 2 else 0
            da = a.step_host_async(bufs[n % 2].data_ptr(), bufs[(n + 1) % 2].data_ptr(), fixed)
            db = b.step_fixed(fixed) if fixed else b.step()
            assert da["iterations"] == db["iterations"], n
        a.wait()
        assert np.array_equal(bufs[1].numpy().view(np.uint64), np.ascontiguousarray(b.get_u()[inner]).view(np.uint64))


@pytest.mark.parametrize("n_slabs", [1, 3])
def test_step_host_async_fallbacks(gpu, n_slabs):
    """step_host_async with pageable numpy buffers (or on a slab group) is step_host: the result
    is on the host when the call returns; wait() is then a no-op."""
    import workloads
    wl = workloads.small((18, 12, 10, 7), seed=29)
    g = gpu.Grid.make(wl.dims, wl.h)
    p = gpu.seg_params(**{**wl.params, "n_steps": 4, "sor_rel_tol": 1e-8, "rescale_radius": 3.0})
    inner = (slice(1, -1),) * 4
    with gpu.Session(g, n_slabs=n_slabs) as a, gpu.Session(g) as b:
        a.prepare(wl.image, wl.rows, p, wl.u0)
        b.prepare(wl.image, wl.rows, p, wl.u0)
        h_in = np.ascontiguousarray(b.get_u()[inner])
        h_out = np.empty_like(h_in)
        for n, fixed in enumerate([0, 5, 0]):
            da = a.step_host_async(h_in.ctypes.data, h_out.ctypes.data, fixed)
            db = b.step_fixed(fixed) if fixed else b.step()
            assert da["iterations"] == db["iterations"], n
            want = np.ascontiguousarray(b.get_u()[inner])
            assert np.array_equal(h_out.view(np.uint64), want.view(np.uint64)), n  # before any wait()
            h_in, h_out = h_out, h_in
        a.wait()


@pytest.mark.parametrize("n_slabs", [1, 3])
def test_fixed_sweep_steps_vs_oracle(gpu, oracle, n_slabs):
    """ss_session_step_fixed (BASELINE config 4's time step) on 1 and 3 slabs against the C
    restatement's no-early-stop loop, which tests/test_fixed_sweeps_cpu.py pins to the
    reference's own fixed-sweep iterate: u bit for bit, the last residual to 1e-12."""
    import math
    import workloads
    from oracle import oracle_py as op
    sys_path_tests = os.path.dirname(os.path.abspath(__file__))
    if sys_path_tests not in sys.path:
        sys.path.insert(0, sys_path_tests)
    from test_fixed_sweeps_cpu import oracle_fixed_steps
    wl = workloads.small((17, 11, 9, 7), seed=5)
    og = op.Grid.make(wl.dims, wl.h)
    p = op.seg_params(**{**wl.params, "n_steps": 2, "sor_rel_tol": 0.0})
    u_or, res = oracle_fixed_steps(oracle, og, wl, p, 2, 9)
    g = gpu.Grid.make(wl.dims, wl.h)
    with gpu.Session(g, n_slabs=n_slabs) as s:
        s.prepare(wl.image, wl.rows, gpu.seg_params(**{**wl.params, "n_steps": 2, "sor_rel_tol": 0.0}), wl.u0)
        d = [s.step_fixed(9) for _ in range(2)]
        u = s.get_u()
    assert [x["iterations"] for x in d] == [9, 9]
    assert np.array_equal(u.view(np.uint64), u_or.view(np.uint64))
    for x, r in zip(d, res):
        assert math.isclose(x["residual"], r, rel_tol=1e-12)


@pytest.mark.parametrize("n_slabs,kernel", [(1, "tma"), (1, "auto"), (3, "tma"), (1, "ldg")])
def test_fixed_sweep_steps_without_diagnostics(gpu, oracle, n_slabs, kernel):
    """step_fixed(diag=False): nobody reads the residual, so the solve runs in SorState::fixed
    mode 2 -- no residual arithmetic and the red pass that would only evaluate the last residual
    stays idle.  u after mixed no-diag / diag steps is the oracle's bit for bit, the diag step
    still reports its own residual, and ss_session_fixed_sweeps (which returns the residual)
    still evaluates it."""
    import math
    import workloads
    from oracle import oracle_py as op
    sys_path_tests = os.path.dirname(os.path.abspath(__file__))
    if sys_path_tests not in sys.path:
        sys.path.insert(0, sys_path_tests)
    from test_fixed_sweeps_cpu import oracle_fixed_steps
    # 40 x 24 rows: enough items for the TMA pass's counter hand-out on one slab
    wl = workloads.small((40, 24, 9, 7), seed=6)
    og = op.Grid.make(wl.dims, wl.h)
    prm = {**wl.params, "n_steps": 3, "sor_rel_tol": 0.0}
    u_or, res = oracle_fixed_steps(oracle, og, wl, op.seg_params(**prm), 3, 9)
    g = gpu.Grid.make(wl.dims, wl.h)
    with gpu.Session(g, n_slabs=n_slabs) as s:
        s.set_kernel(kernel)
        s.prepare(wl.image, wl.rows, gpu.seg_params(**prm), wl.u0)
        assert s.step_fixed(9, diag=False) is None
        assert s.step_fixed(9, diag=False) is None
        d = s.step_fixed(9)
        u = s.get_u()
        r_fs = s.fixed_sweeps(4)  # assemble + 4 sweeps, returns the 4th iteration's residual
        s.profile()
        s.step_fixed(5, diag=False)
        sweeps = s.profile()["sweeps"]
    assert np.array_equal(u.view(np.uint64), u_or.view(np.uint64))
    assert d["iterations"] == 9 and math.isclose(d["residual"], res[2], rel_tol=1e-12)
    assert r_fs > 0.0 and math.isfinite(r_fs)
    assert sweeps == 5


def test_kernel_switch_within_a_session(gpu):
    """ss_session_set_kernel between solves of ONE session (the captured CUDA
    graph was keyed without the item shape, so a switch between the whole-row and the
    2D-tiled TMA passes could replay the old graph): every solve runs -- and reports -- the
    kernel asked for, and all give the same iterate."""
    import workloads
    wl = workloads.small((40, 12, 10, 6), seed=9)
    g = gpu.Grid.make(wl.dims, wl.h)
    p = gpu.seg_params(**{**wl.params, "n_steps": 8, "sor_rel_tol": 1e-8})
    outs = {}
    with gpu.Session(g) as s:
        s.prepare(wl.image, wl.rows, p, wl.u0)
        u_start = s.get_u()
        for kernel in ("tma", "tma2d", "tma", "ldg", "tma2d", "resident", "tma"):
            s.set_u(u_start)
            s.set_kernel(kernel)
            d = s.step()
            assert s.sor_kernel() == kernel
            outs.setdefault(kernel, []).append((d["iterations"], s.get_u()))
    its0, u0 = outs["tma"][0]
    for kernel, runs in outs.items():
        for its, u in runs:
            assert its == its0, kernel
            assert np.array_equal(u.view(np.uint64), u0.view(np.uint64)), kernel
