"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the oracle restatement, bit for bit.

The reference's arithmetic is deterministic per doxel and red-black SOR is
order-independent within a colour phase, so with -fmad=false and the
reference's expression order the iterates are *identical*, which is stronger
than north_star's max|du| <= 1e-6 per step.  Only the residual value (a sum in
a different order) may differ in the last bits; tests allow 1e-12 relative on
it and require identical iteration counts.
"""
import os

import numpy as np
import pytest

import _cases as cs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
pytestmark = pytest.mark.gpu


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def G_of(ss, d):
    return ss.Grid.make(tuple(int(x) for x in d["dims"]), float(d["h"]))


def assert_bits(a, b, what):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, what
    diff = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64)) if a.dtype == np.float64 else \
        np.flatnonzero(a != b)
    assert diff.size == 0, f"{what}: {diff.size} of {a.size} differ, first at {diff[:5]}"


# ------------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("tag", ["a", "b"])
def test_assemble_golden(gpu, tag):
    d = load(f"assemble_sor_{tag}")
    g = G_of(gpu, d)
    c = gpu.assemble_step(d["u"], d["G"], float(d["tau"]), float(d["eps"]), g)
    assert_bits(c.offdiag, d["off"], "offdiag")
    assert_bits(c.diag, d["diag"], "diag")
    assert_bits(c.abar, d["abar"], "abar")
    c0 = gpu.assemble_step(d["u"], None, float(d["tau"]), float(d["eps"]), g)
    assert_bits(c0.offdiag, d["off_noG"], "offdiag G=1")
    assert_bits(c0.diag, d["diag_noG"], "diag G=1")


@pytest.mark.parametrize("tag", ["a", "b"])
def test_sor_golden(gpu, tag):
    d = load(f"assemble_sor_{tag}")
    g = G_of(gpu, d)
    r = gpu.redblack_sor(d["off"], d["u"], d["u"], float(d["omega"]), float(d["tol"]), 500, g)
    assert r.iterations == int(d["sor_iters"])
    assert abs(r.residual - float(d["sor_res"])) <= 1e-12 * float(d["sor_res"])
    assert_bits(r.u, d["sor_u"], "sor u")


def test_preprocess_golden(gpu):
    d = load("preprocess")
    g = G_of(gpu, d)
    sig = np.sqrt(2) * 0.25
    I0s = gpu.heat_smooth(d["image"], g, sig, 1)
    assert_bits(I0s, d["I0s"], "heat_smooth(image)")
    th = gpu.local_threshold(d["image"], d["rows"], g, 0.5, 0.0)
    assert_bits(th, d["threshold"], "local_threshold")
    ITs = gpu.heat_smooth(th, g, sig, 2)
    assert_bits(ITs, d["ITs"], "heat_smooth(threshold), 2 steps")
    G = gpu.face_coefficients(d["I0s"], d["ITs"], float(d["K"]), float(d["delta"]),
                              float(d["vartheta"]), g)
    assert_bits(G, d["G"], "face_coefficients")


def test_seedinit_golden(gpu):
    d = load("seedinit")
    g = G_of(gpu, d)
    assert_bits(gpu.build_initial(d["rows"], g, 1.0, 3.0, 0), d["u0_peak"], "build_initial peak")
    assert_bits(gpu.build_initial(d["rows"], g, 0.5, 2.5, 1), d["u0_linear"], "build_initial linear")
    assert_bits(gpu.local_rescale(d["noisy"], d["rows"], g), d["rescale_rowradius"], "rescale rows")
    assert_bits(gpu.local_rescale(d["noisy"], d["rows"], g, 2.2), d["rescale_r22"], "rescale r=2.2")


def _seg_params(ss, h, **kw):
    return ss.seg_params(tau=h, epsilon=1e-3, omega=1.4, n_steps=3, sigma=np.sqrt(2) * h, K=200.0,
                         delta=0.5, vartheta=0.5, rescale_radius=3.0, **kw)


def test_segment_golden(gpu):
    d = load("segment")
    g = G_of(gpu, d)
    h = float(d["h"])
    u, diags = gpu.segment(d["image"], d["rows"], _seg_params(gpu, h, sor_tol=1e-9), g)
    assert [x["iterations"] for x in diags] == list(d["iters"])
    assert_bits(u, d["u"], "segment u (absolute tol)")
    u2, diags2 = gpu.segment(d["image"], d["rows"], _seg_params(gpu, h, sor_rel_tol=1e-8), g)
    assert [x["iterations"] for x in diags2] == list(d["iters_rel"])
    np.testing.assert_allclose([x["tol"] for x in diags2], d["tol_rel"], rtol=1e-13)
    assert_bits(u2, d["u_rel"], "segment u (relative tol)")


def test_session_matches_segment(gpu):
    d = load("segment")
    g = G_of(gpu, d)
    h = float(d["h"])
    p = _seg_params(gpu, h, sor_rel_tol=1e-8)
    for mode in (0, 1):
        with gpu.Session(g) as s:
            s.set_loop_mode(mode)
            s.prepare(d["image"], d["rows"], p)
            its = [s.step()["iterations"] for _ in range(3)]
            assert its == list(d["iters_rel"]), mode
            assert_bits(s.get_u(), d["u_rel"], f"session u, loop mode {mode}")
            mask = s.get_mask(0.5)
            ref_mask = (d["u_rel"][g.interior] >= 0.5).astype(np.uint8)
            assert_bits(mask, ref_mask, "mask")


def test_eoc_golden(gpu):
    """eoc.cpp:83-137 driven through the per-call API: Table 1 rows n=10, 20."""
    d = load("eoc")
    for n, key, paper in [(10, "e10", 1.680403e-2), (20, "e20", 4.653133e-3)]:
        err = eoc_row_gpu(gpu, n)
        assert err == pytest.approx(float(d[key]), rel=1e-12)
        assert abs(err - paper) / paper < 0.05  # tests/test_eoc.cpp:129-132


def exact_u(x0, x1, x2, x3, t):
    return (x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3 - 1.0) / 6.0 + t


def eoc_row_gpu(ss, n, omega=1.5, tol=1e-8):
    steps = {10: 1, 20: 4, 40: 16, 80: 64, 160: 256}[n]
    dmin, dmax, T = -1.25, 1.25, 0.0625
    h = (dmax - dmin) / n
    tau = T / steps
    g = ss.Grid.make((n,) * 4, h)
    x = dmin + (np.arange(n + 2) - 0.5) * h
    L, K, J, I = np.meshgrid(x, x, x, x, indexing="ij")

    def full(t):
        return exact_u(I, J, K, L, t)

    u = full(0.0)
    ghost = np.ones(g.shape, bool)
    ghost[g.interior] = False
    err_sq = 0.0
    for step in range(1, steps + 1):
        t = step * tau
        c = ss.assemble_step(u, None, tau, h * h, g)
        u = u.copy()
        u[ghost] = full(t)[ghost]
        r = ss.redblack_sor(c, u, u, omega, tol, 10000, g)
        u = r.u
        e = (u - full(t))[g.interior]
        step_sum = 0.0
        for l in range(n):
            step_sum += float(np.sum(e[l] ** 2))
        err_sq += tau * h ** 4 * step_sum
    return np.sqrt(err_sq)


# ------------------------------------------------------------------ oracle, random cases
SHAPES = [(6, 5, 4, 5), (7, 3, 5, 4), (1, 4, 3, 5), (9, 1, 1, 3), (33, 6, 5, 4), (64, 3, 2, 3),
          (257, 5, 9, 3), (130, 17, 10, 2)]  # wide rows: R < 8 rows per item, several slots per lane


@pytest.mark.parametrize("dims", SHAPES)
def test_assemble_and_sor_random(gpu, oracle, dims):
    g = gpu.Grid.make(dims, (0.3, 0.25, 0.5, 0.2))
    og = cs.grid(dims, (0.3, 0.25, 0.5, 0.2))
    u = cs.rand_field(dims, sum(dims), ghosts="random")
    G = cs.rand_G(dims, 7 + sum(dims))
    st, off, dg, ab = oracle.assemble_step(og, u, G, 0.07, 2e-3)
    assert st == 0
    c = gpu.assemble_step(u, G, 0.07, 2e-3, g)
    assert_bits(c.offdiag, off, "offdiag")
    assert_bits(c.diag, dg, "diag")
    assert_bits(c.abar, ab, "abar")
    rhs = cs.rand_field(dims, 99)
    st, uo, it, res = oracle.redblack_sor(og, off, rhs, u, 1.3, 1e-12, 2000)
    assert st == 0
    r = gpu.redblack_sor(c, rhs, u, 1.3, 1e-12, 2000, g)
    assert r.iterations == it
    assert r.residual == pytest.approx(res, rel=1e-12)
    assert_bits(r.u, uo, "sor u")


def test_sor_noconvergence_is_solver_error(gpu, oracle):
    dims = (8, 6, 5, 4)
    g = gpu.Grid.make(dims, 0.1)
    og = cs.grid(dims, 0.1)
    u = cs.rand_field(dims, 3)
    st, off, _, _ = oracle.assemble_step(og, u, None, 5.0, 1e-3)
    st, uo, it, res = oracle.redblack_sor(og, off, u, u, 1.2, 1e-300, 7)
    assert st == oracle_noconv()
    with pytest.raises(gpu.SolverError) as e:
        gpu.redblack_sor(off, u, u, 1.2, 1e-300, 7, g)
    assert e.value.iterations == 7 == it
    assert e.value.last_residual == pytest.approx(res, rel=1e-12)


def oracle_noconv():
    from oracle import oracle_py
    return oracle_py.ERR_NOCONVERGE


def test_nonfinite_is_numerical_error(gpu):
    dims = (4, 4, 3, 3)
    g = gpu.Grid.make(dims, 0.5)
    u = cs.rand_field(dims, 5)
    u[2, 2, 2, 2] = np.inf
    with pytest.raises(gpu.NumericalError):
        gpu.assemble_step(u, None, 0.1, 1e-3, g)


def test_validation_errors(gpu):
    dims = (4, 4, 3, 3)
    g = gpu.Grid.make(dims, 0.5)
    u = cs.rand_field(dims, 5)
    with pytest.raises(gpu.ValidationError):
        gpu.assemble_step(u, None, 0.1, 0.0, g)      # epsilon must be > 0
    with pytest.raises(gpu.ValidationError):
        gpu.redblack_sor(np.zeros(g.shape + (8,)), u, u, 2.0, 1e-8, 10, g)  # omega in (0,2)
    with pytest.raises(gpu.ValidationError):
        gpu.local_threshold(u, [(5, 1, 1, 1, 1.0)], g)  # frame out of range
    with pytest.raises(gpu.ValidationError):
        gpu.face_coefficients(u, u, 1.0, 1.5, 0.0, g)  # delta in [0,1]


def test_heat_assembly_bits(gpu, oracle):
    dims = (5, 4, 6, 3)
    g = gpu.Grid.make(dims, (0.2, 0.3, 0.25, 0.5))
    og = cs.grid(dims, (0.2, 0.3, 0.25, 0.5))
    st, off, dg, ab = oracle.assemble_heat_step(og, 0.013)
    c = gpu.assemble_heat_step(g, 0.013)
    assert_bits(c.offdiag, off, "heat off")
    assert_bits(c.diag, dg, "heat diag")
    assert_bits(c.abar, ab, "heat abar")


@pytest.mark.parametrize("dims", [(7, 6, 5, 4), (12, 9, 8, 3)])
def test_balls_random(gpu, oracle, dims):
    g = gpu.Grid.make(dims, 1.0)
    og = cs.grid(dims, 1.0)
    rng = np.random.default_rng(sum(dims))
    rows = [(int(rng.integers(0, dims[3])), rng.uniform(0, dims[0] - 1), rng.uniform(0, dims[1] - 1),
             rng.uniform(0, dims[2] - 1), rng.uniform(0.8, 3.5)) for _ in range(40)]
    img = cs.rand_field(dims, 1)
    st, th = oracle.local_threshold(og, img, rows, 0.3, -1.0)
    assert st == 0
    assert_bits(gpu.local_threshold(img, rows, g, 0.3, -1.0), th, "threshold, 40 balls")
    st, rs = oracle.local_rescale(og, img, rows, None)
    assert_bits(gpu.local_rescale(img, rows, g), rs, "rescale, 40 balls")
    st, u0 = oracle.build_initial(og, rows, 0.7, 2.2, 0)
    assert_bits(gpu.build_initial(rows, g, 0.7, 2.2, 0), u0, "initial, 40 balls")
    st, m = 0, oracle.extract_mask(og, rs, 0.5)
    assert_bits(gpu.extract_mask(rs, g, 0.5), m, "mask")


def test_empty_ball_rejected(gpu):
    dims = (6, 6, 6, 2)
    g = gpu.Grid.make(dims, 1.0)
    img = cs.rand_field(dims, 1)
    # radius 0.2 around a non-lattice point covers no doxel (preprocess.cpp:89-91)
    with pytest.raises(gpu.ValidationError, match="row 2"):
        gpu.local_threshold(img, [(0, 2, 2, 2, 1.0), (1, 2.5, 2.5, 2.5, 0.2)], g)


def test_fixed_sweeps_and_launch_count(gpu):
    d = load("segment")
    g = G_of(gpu, d)
    h = float(d["h"])
    with gpu.Session(g) as s:
        s.prepare(d["image"], d["rows"], _seg_params(gpu, h, sor_rel_tol=1e-8))
        s.set_kernel("tma")
        n0 = gpu.launch_count()
        r = s.fixed_sweeps(50)
        assert np.isfinite(r)
        assert gpu.launch_count() - n0 >= 100  # 50 x (red, black with the finalize in its head)
        s.set_kernel("wave")
        n0 = gpu.launch_count()
        s.fixed_sweeps(50)
        assert gpu.launch_count() - n0 >= 75  # 25 x (wavefront, finalize, finalize)


def test_grid_helpers(gpu, oracle):
    dims = (7, 5, 4, 3)
    g = gpu.Grid.make(dims, 0.5)
    og = cs.grid(dims, 0.5)
    f = cs.rand_field(dims, 17)
    assert_bits(gpu.apply_mirror_ghosts(f, g), oracle.apply_mirror_ghosts(og, f), "mirror ghosts")
    d = gpu.apply_dirichlet(f, g, 0.25)
    ghost = np.ones(g.shape, bool)
    ghost[g.interior] = False
    assert np.all(d[ghost] == 0.25) and np.array_equal(d[~ghost], f[~ghost])
    lo, hi = gpu.interior_minmax(f, g)
    assert lo == f[g.interior].min() and hi == f[g.interior].max()


def test_per_call_api_thread_safe(gpu):
    """The per-call entry points share one cached device context: concurrent calls from
    several host threads (ctypes drops the GIL) on different grids give the serial results."""
    import threading
    cases = []
    for dims in [(6, 5, 4, 5), (9, 7, 3, 4)]:
        g = gpu.Grid.make(dims, 0.25)
        u = cs.rand_field(dims, sum(dims))
        G = cs.rand_G(dims, 3 + sum(dims))
        cases.append((g, u, G, gpu.assemble_step(u, G, 0.1, 1e-3, g)))
    errors = []

    def work(k):
        try:
            for r in range(4):
                g, u, G, want = cases[(k + r) % 2]
                got = gpu.assemble_step(u, G, 0.1, 1e-3, g)
                for f in ("offdiag", "diag", "abar"):
                    assert np.array_equal(getattr(got, f), getattr(want, f))
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("kernel", ["auto", "tma", "ldg", "resident"])
def test_segment_step_noconvergence(gpu, oracle, kernel):
    """segment()'s SOR hitting sor_max_iter raises SolverError with the reference's
    iteration count and last residual (solver.cpp:391-395), from every SOR kernel."""
    d = load("segment")
    g = G_of(gpu, d)
    h = float(d["h"])
    kw = dict(tau=h, epsilon=1e-3, omega=1.4, n_steps=1, sigma=np.sqrt(2) * h, K=200.0, delta=0.5,
              vartheta=0.5, rescale_radius=3.0, sor_tol=1e-300, sor_max_iter=9)
    from oracle.oracle_py import Grid as OG, seg_params as osp
    st, _, info = oracle.segment(OG.make(tuple(int(x) for x in d["dims"]), h), d["image"], d["rows"], osp(**kw))
    assert st == oracle_noconv()
    with gpu.Session(g) as s:
        s.set_kernel(kernel)
        s.prepare(d["image"], d["rows"], gpu.seg_params(**kw))
        with pytest.raises(gpu.SolverError) as e:
            s.step()
    assert e.value.iterations == 9
    assert e.value.last_residual > 0


@pytest.mark.parametrize("k", [5, 12, 23])
def test_stopping_tie_at_the_references_own_residual(gpu, ref, k):
    """the stopping residual is a sum of squares in a different order than the
    reference's (256-lane trees of per-slice partials vs its sequential sweep,
    solver.cpp:306-312, :357-359), so it can differ from the reference's in the last bits.
    With sor_tol set to the reference's own residual after k iterations the reference stops
    at k (res <= tol); this documents how the GPU decides the tie: at k when its residual is
    not above the tolerance, else one iteration later -- and the residuals agree to 1e-12."""
    dims = (9, 7, 6, 5)
    g = gpu.Grid.make(dims, 0.125)
    og = cs.grid(dims, 0.125)
    u = cs.rand_field(dims, 40 + k)
    st, off, _, _ = ref.assemble_step(og, u, None, 0.2, 1e-3)
    st, _, it, r_k = ref.redblack_sor(og, off, u, u, 1.4, 1e-300, k)
    assert st == oracle_noconv() and it == k
    st, u_ref, it_ref, res_ref = ref.redblack_sor(og, off, u, u, 1.4, r_k, 10 * k)
    assert st == 0 and it_ref == k and res_ref == r_k  # the reference: res <= tol at k
    with pytest.raises(gpu.SolverError) as e:  # the GPU's own residual after exactly k sweeps
        gpu.redblack_sor(off, u, u, 1.4, 1e-300, k, g)
    r_gpu = e.value.last_residual
    assert r_gpu == pytest.approx(r_k, rel=1e-12)
    r = gpu.redblack_sor(off, u, u, 1.4, r_k, 10 * k, g)
    assert r.iterations == (k if r_gpu <= r_k else k + 1)
    if r.iterations == k:
        assert_bits(r.u, u_ref, "tie decided at k: the reference's iterate")


@pytest.mark.parametrize("mode", ["step", "step_fixed", "fixed_sweeps", "step_host"])
def test_session_nonfinite_is_numerical_error(gpu, mode):
    """assemble_step's NumericalError (solver.cpp:71-75) from every session step flavour --
    decided on the device (sor_init reads the assembly flag), no host sync in between; the
    session's u is left as it was (fixed_sweeps used to skip the check)."""
    import workloads
    wl = workloads.small((12, 10, 8, 6), seed=3)
    g = gpu.Grid.make(wl.dims, wl.h)
    with gpu.Session(g) as s:
        s.prepare(wl.image, wl.rows, gpu.seg_params(**{**wl.params, "n_steps": 3}), wl.u0)
        u = s.get_u()
        u[3, 4, 5, 6] = np.nan
        s.set_u(u)
        with pytest.raises(gpu.NumericalError):
            if mode == "step":
                s.step()
            elif mode == "step_fixed":
                s.step_fixed(5)
            elif mode == "fixed_sweeps":
                s.fixed_sweeps(5)
            else:
                s.step_host(np.ascontiguousarray(u[1:-1, 1:-1, 1:-1, 1:-1]), None, 0)
        after = s.get_u()
        assert np.array_equal(np.isnan(after), np.isnan(u)) and np.array_equal(after[~np.isnan(u)], u[~np.isnan(u)])


def test_explicit_zero_rescale_radius(gpu, oracle):
    """rescale_radius = 0 set explicitly is the reference's r = 0 ball (<= 1 doxel: a no-op,
    seedinit.cpp:73-88), not "each row's own radius"; NaN / None is std::nullopt."""
    from oracle import oracle_py as op
    dims, h = (10, 8, 7, 6), 0.125
    g = gpu.Grid.make(dims, h)
    og = cs.grid(dims, h)
    u = cs.rand_field(dims, 8)
    rows = [(f, 4.0, 3.0, 3.0, 2.5) for f in range(dims[3])]
    assert_bits(gpu.local_rescale(u, rows, g, 0.0), u, "r = 0: no-op")
    assert_bits(gpu.local_rescale(u, rows, g, None), oracle.local_rescale(og, u, rows, None)[1], "per row")
    img = cs.f32_image(dims, 9)
    for rr in (0.0, None):
        kw = dict(tau=h, epsilon=1e-3, omega=1.4, sor_tol=1e-9, n_steps=2, sigma=0.17, K=200.0, delta=0.5,
                  vartheta=0.5, rescale_radius=rr)
        u_g, _ = gpu.segment(img, rows, gpu.seg_params(**kw), g)
        st, u_o, _ = oracle.segment(op.Grid.make(dims, h), img, rows, op.seg_params(**kw))
        assert st == 0
        assert_bits(u_g, u_o, f"segment rescale_radius={rr}")


def test_rsqrt_approximation_bound(gpu):
    """The assembly tail's exactness argument (assemble_tile.cu): q' from rsqrt.approx.f64 +
    two Newton steps lies within ~20 double ulps of the reference's quotient, and a float
    rounding decision is trusted only >= 512 ulps from a midpoint.  That needs the hardware
    approximation's relative error eps0 well below 2^-11 -- checked exhaustively here over every
    normal positive input high word (the only part MUFU.RSQ64H reads)."""
    import ctypes as C
    e = C.c_double(0.0)
    assert gpu.library().ss_selftest_rsqrt(C.byref(e)) == 0
    assert 0.0 < e.value < 2.0 ** -11, e.value
    print("rsqrt.approx.f64 max relative error", e.value)


@pytest.mark.parametrize("case", ["iso_pow2", "iso_pow2_guard", "aniso_pow2", "non_pow2"])
def test_tile_assembly_coefficients_vs_oracle(gpu, oracle, case):
    """The device path's assembly (assemble_tile.cu: TMA-staged bricks, the rsqrt tail with
    its exact fallback, the scaled face gradients behind the range guard) against the oracle's
    assemble_step off-diagonals, bit for bit, on u with a wide range of magnitudes and exact
    zeros.  K = 0 makes the session's G exactly 1 (edge.cpp: 1 / (1 + 0)), so the oracle runs
    with G == 1.  iso_pow2: the scaled path; iso_pow2_guard: one value of 1e-200 trips the
    guard (reference expression); aniso_pow2 / non_pow2: the per-axis expressions."""
    from oracle import oracle_py as op
    dims = (37, 13, 11, 7)
    h = {"iso_pow2": 1 / 32, "iso_pow2_guard": 1 / 32, "aniso_pow2": (1 / 32, 1 / 16, 1 / 32, 1 / 64),
         "non_pow2": (0.1, 0.07, 0.13, 0.05)}[case]
    g = gpu.Grid.make(dims, h)
    og = op.Grid.make(dims, h)
    tau, eps = 0.03, 1e-3
    img = cs.f32_image(dims, 7)
    rows = [(f, 18.0, 6.0, 5.0, 3.0) for f in range(dims[3])]
    rng = np.random.default_rng(77)
    u = np.zeros(g.shape)
    vals = rng.normal(0.5, 0.4, size=u[1:-1, 1:-1, 1:-1, 1:-1].shape) * 10.0 ** rng.uniform(-3, 3, size=u[1:-1, 1:-1, 1:-1, 1:-1].shape)
    vals[rng.random(vals.shape) < 0.2] = 0.0
    u[1:-1, 1:-1, 1:-1, 1:-1] = vals
    if case == "iso_pow2_guard":
        u[3, 4, 5, 6] = 1e-200
    p = gpu.seg_params(tau=tau, epsilon=eps, omega=1.4, sor_tol=1e-9, n_steps=1, sigma=0.1, K=0.0, delta=0.5,
                       vartheta=0.5, rescale_radius=2.0)
    with gpu.Session(g) as s:
        s.prepare(img, rows, p, None)
        s.set_u(u)
        off_gpu = s.assemble_export()
    st, off_ref, _, _ = oracle.assemble_step(og, u, None, tau, eps)
    assert st == 0
    assert_bits(off_gpu, off_ref, f"tile assembly, {case}")


def _cert_field(dims, seed, sharp, scale=1.0):
    """u in [0, 1] as segmentation iterates are: a smooth 4D profile (or, sharp, a ball with a
    one-doxel edge: gradients ~ 1/h) plus noise, Dirichlet ghosts 0 (the reference's setting);
    scale != 1: affinely spread to [-scale, scale] (a larger max |u|: a wider certified margin)."""
    rng = np.random.default_rng(seed)
    n1, n2, n3, n4 = dims
    l, k, j, i = np.meshgrid(*[np.arange(n) for n in dims[::-1]], indexing="ij")
    r = np.sqrt(((i - n1 / 2) / n1) ** 2 + ((j - n2 / 2) / n2) ** 2 + ((k - n3 / 2) / n3) ** 2
                + ((l - n4 / 2) / n4) ** 2)
    prof = (r < 0.3).astype(float) if sharp else 1.0 / (1.0 + 8.0 * r)
    u = np.zeros(cs.shape(dims))
    u[1:-1, 1:-1, 1:-1, 1:-1] = np.clip(prof + rng.normal(0, 0.02, prof.shape), 0.0, 1.0)
    if scale != 1.0:
        u[1:-1, 1:-1, 1:-1, 1:-1] = (2.0 * u[1:-1, 1:-1, 1:-1, 1:-1] - 1.0) * scale
    return u


def _assemble_session(gpu, g, u, tau, eps):
    dims = (g.n1, g.n2, g.n3, g.n4)
    img = cs.f32_image(dims, 7)
    rows = [(f, dims[0] / 2, dims[1] / 2, dims[2] / 2, 3.0) for f in range(dims[3])]
    p = gpu.seg_params(tau=tau, epsilon=eps, omega=1.4, sor_tol=1e-9, n_steps=1, sigma=0.1, K=0.0, delta=0.5,
                       vartheta=0.5, rescale_radius=2.0)
    with gpu.Session(g) as s:
        s.prepare(img, rows, p, None)
        s.set_u(u)
        return s.assemble_export()


@pytest.mark.parametrize("h,sharp,scale", [(1 / 32, False, 1.0), (1 / 64, False, 1.0), (1 / 32, True, 1.0),
                                           (1 / 128, True, 1.0), (1 / 32, False, 2.0), (1 / 16, True, 3.0)])
def test_certified_face_gradients_vs_oracle(gpu, oracle, h, sharp, scale, monkeypatch):
    """The certified face gradients (assemble_tile.cu face_sq_cert: central differences instead
    of the reference's rounded corner sums, within a proven bound of its |grad_f u|^2, the float
    rounding decision trusted only outside that bound) give the reference's coefficients bit for
    bit on ~0.9 M doxels (7 M faces) of u in [0, 1], smooth and with sharp edges, at h = 1/32,
    1/64, 1/128; so do the exact scaled gradients (SSB_ASM_CERT=0).  With no margin
    (SSB_ASM_CERT=2, test-only) some coefficients must come out wrong: the path under test is the
    one that ran, and its margin is what keeps it exact."""
    from oracle import oracle_py as op
    dims = (64, 30, 24, 20)
    g = gpu.Grid.make(dims, h)
    tau, eps = h, 1e-3
    u = _cert_field(dims, 11 + int(sharp), sharp, scale)
    st, off_ref, _, _ = oracle.assemble_step(op.Grid.make(dims, h), u, None, tau, eps)
    assert st == 0
    monkeypatch.setenv("SSB_ASM_CERT", "1")
    assert_bits(_assemble_session(gpu, g, u, tau, eps), off_ref, f"certified gradients h={h} sharp={sharp}")
    monkeypatch.setenv("SSB_ASM_CERT", "0")
    assert_bits(_assemble_session(gpu, g, u, tau, eps), off_ref, f"exact scaled gradients h={h} sharp={sharp}")
    if not sharp and h == 1 / 64 and scale == 1.0:
        monkeypatch.setenv("SSB_ASM_CERT", "2")
        off_bad = _assemble_session(gpu, g, u, tau, eps)
        wrong = int(np.count_nonzero(off_bad.view(np.uint64) != off_ref.view(np.uint64)))
        print(f"no-margin certified gradients: {wrong} of {off_ref.size} coefficients differ")
        assert wrong > 0


@pytest.mark.parametrize("case", ["iso_pow2", "iso_pow2_guard", "iso_pow2_exact", "aniso_pow2", "non_pow2"])
def test_tile_face_coefficients_vs_oracle(gpu, oracle, case, monkeypatch):
    """The device path's edge detector (assemble_tile.cu edge_tile_kernel: TMA-staged I0s / ITs
    bricks; on isotropic power-of-two grids the scaled face gradients |grad_f I| = c sqrt(S)
    behind the range guard over both images) against the oracle's face_coefficients, bit for
    bit, on images with magnitudes 1e-3..1e3 and exact zeros.  iso_pow2: the scaled path (two
    guard launches more than with SSB_EDGE_SCALED=0, iso_pow2_exact); iso_pow2_guard: one value
    of 1e-200 in ITs trips the guard (the reference's expression runs)."""
    from oracle import oracle_py as op
    dims = (37, 13, 11, 7)
    h = {"iso_pow2": 1 / 32, "iso_pow2_guard": 1 / 32, "iso_pow2_exact": 1 / 64,
         "aniso_pow2": (1 / 32, 1 / 16, 1 / 32, 1 / 64), "non_pow2": (0.1, 0.07, 0.13, 0.05)}[case]
    g = gpu.Grid.make(dims, h)
    rng = np.random.default_rng(5)
    I0 = rng.normal(0.5, 0.3, size=g.shape) * 10.0 ** rng.uniform(-3, 3, size=g.shape)
    I0[rng.random(g.shape) < 0.15] = 0.0
    IT = np.clip(rng.normal(0.5, 0.4, size=g.shape), 0.0, 1.0)
    if case == "iso_pow2_guard":
        IT[2, 3, 4, 5] = 1e-200
    monkeypatch.setenv("SSB_EDGE_SCALED", "0" if case == "iso_pow2_exact" else "1")
    K, delta, vartheta = 1000.0, 0.5, 0.5
    gpu.face_coefficients(I0, IT, K, delta, vartheta, g)  # the grid's cached domain is built here
    n0 = gpu.launch_count()
    G = gpu.face_coefficients(I0, IT, K, delta, vartheta, g)
    n_scaled = gpu.launch_count() - n0
    st, G_ref = oracle.face_coefficients(op.Grid.make(dims, h), I0, IT, K, delta, vartheta)
    assert st == 0
    assert_bits(G, G_ref, f"tile face_coefficients, {case}")
    if case in ("iso_pow2", "iso_pow2_exact"):
        monkeypatch.setenv("SSB_EDGE_SCALED", "0")
        n0 = gpu.launch_count()
        G0 = gpu.face_coefficients(I0, IT, K, delta, vartheta, g)
        n_exact = gpu.launch_count() - n0
        assert_bits(G0, G_ref, f"tile face_coefficients, {case}, exact gradients")
        assert n_scaled - n_exact == (2 if case == "iso_pow2" else 0), (n_scaled, n_exact)
