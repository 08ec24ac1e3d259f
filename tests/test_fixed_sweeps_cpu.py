"""CPU: the fixed-sweep parity pin (BASELINE config 4) and the pins file.

The reference has no fixed-sweep mode: redblack_sor throws SolverError at max_iter
and drops the iterate (solver.cpp:201-206, :391-395).  tests/golden/make_pins.py
recovers the reference's own iterate after exactly n sweeps with a second call at
sor_tol = the thrown residual (oracle/ref_shim.cpp ref_segment_fixed, mode 0).  Here
that recovery is checked against the oracle restatement, whose redblack_sor returns
its last iterate on non-convergence -- bit for bit over whole time steps -- and the
explicit rescale radius semantics (std::optional engaged with r <= 0) are pinned.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import _cases as cs

HERE = os.path.dirname(os.path.abspath(__file__))


def same_bits(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def oracle_fixed_steps(oracle, g, wl, p, n_steps, n_sweeps):
    """segment() preamble + n_steps of (assemble, exactly n_sweeps sweeps, rescale) on the oracle."""
    rr = None if math.isnan(p.rescale_radius) else p.rescale_radius
    st, u = oracle.local_rescale(g, wl.u0, wl.rows, rr)
    assert st == 0
    st, th = oracle.local_threshold(g, wl.image, wl.rows, p.lambda_, p.background)
    assert st == 0
    sm = (p.sigma, p.smooth_steps, p.smooth_omega, p.smooth_tol, p.smooth_max_iter)
    st, I0s = oracle.heat_smooth(g, wl.image, *sm)
    assert st == 0
    st, ITs = oracle.heat_smooth(g, th, *sm)
    assert st == 0
    st, G = oracle.face_coefficients(g, I0s, ITs, p.K, p.delta, p.vartheta)
    assert st == 0
    res = []
    for _ in range(n_steps):
        st, off, _, _ = oracle.assemble_step(g, u, G, p.tau, p.epsilon)
        assert st == 0
        st, u, it, r = oracle.redblack_sor(g, off, u, u, p.omega, 1e-300, n_sweeps)
        assert st == 2 and it == n_sweeps  # OR_ERR_NOCONVERGE, iterate kept
        res.append(r)
        st, u = oracle.local_rescale(g, u, wl.rows, rr)
        assert st == 0
    return u, res


@pytest.mark.parametrize("dims,n_sweeps", [((16, 12, 10, 8), 7), ((13, 9, 7, 5), 12)])
def test_fixed_sweep_pin_matches_oracle(oracle, ref, dims, n_sweeps):
    import workloads
    from oracle import oracle_py as op
    wl = workloads.small(dims)
    g = op.Grid.make(wl.dims, wl.h)
    p = op.seg_params(**{**wl.params, "n_steps": 2, "sor_rel_tol": 0.0})
    st, u_ref, info = ref.segment_fixed(g, wl.image, wl.rows, p, wl.u0, 3, n_sweeps, 0)
    assert st == 0, ref.lib.ref_last_error()
    u_or, res = oracle_fixed_steps(oracle, g, wl, p, 2, n_sweeps)
    assert same_bits(u_ref, u_or)
    assert [d["iterations"] for d in info["diags"]] == [n_sweeps] * 2
    np.testing.assert_allclose([d["residual"] for d in info["diags"]], res, rtol=1e-12)
    # bench mode (1): the same work, u not advanced (the reference drops the iterate)
    st, u_b, info_b = ref.segment_fixed(g, wl.image, wl.rows, p, wl.u0, 3, n_sweeps, 1)
    assert st == 0 and [d["iterations"] for d in info_b["diags"]] == [n_sweeps] * 2


@pytest.mark.parametrize("radius", [0.0, -1.5, 0.4])
def test_explicit_small_rescale_radius(oracle, ref, radius):
    """rescale_radius set to <= 0 (or < 1 voxel) is an explicit radius, not "per row":
    the ball holds at most one doxel, hi > lo fails and the rescale is a no-op
    (seedinit.cpp:73-88) -- ADVICE r01."""
    dims = (6, 5, 4, 5)
    g = cs.grid(dims, 0.25)
    u = cs.rand_field(dims, 31)
    rows = cs.centers_overlapping(dims)
    st, a = oracle.local_rescale(g, u, rows, radius)
    st2, b = ref.local_rescale(g, u, rows, radius)
    assert st == 0 and st2 == 0 and same_bits(a, b) and same_bits(a, u)
    st, c = oracle.local_rescale(g, u, rows, None)  # std::nullopt: each row's own radius
    st2, d = ref.local_rescale(g, u, rows, None)
    assert same_bits(c, d) and not same_bits(c, u)


def test_pins_file_consistent():
    pins = json.load(open(os.path.join(HERE, "golden", "pins.json")))
    for name in ("config0", "config1", "config2", "config4"):
        assert name in pins, name
        pin = pins[name]
        for k in ("iterations", "residual", "tol", "umin", "umax"):
            assert len(pin[k]) == pin["steps"], (name, k)
        assert len(pin["u_sha256"]) == 64 and pin["mask_voxels"] > 0
    assert pins["config4"]["iterations"] == [50] * pins["config4"]["steps"]
    # the cheapest config's inputs regenerate bit for bit on this host too
    import workloads
    wl = workloads.config0()
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(wl.image) == pins["config0"]["inputs"]["image"]
    assert sha(wl.u0) == pins["config0"]["inputs"]["u0"]
