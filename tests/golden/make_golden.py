"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref was
compiled from it by oracle/Makefile):

    python tests/golden/make_golden.py

Every fixture stores the inputs and the reference's outputs of one public
reference call on a small seeded case.  The oracle restatement and the CUDA
path are both checked against these bit for bit (tests/test_oracle_pin.py,
tests/test_gpu_parity.py); the fixtures travel to the GPU box, the reference
does not.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle_py as op  # noqa: E402
import _cases as cs  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    print("wrote", name, {k: np.shape(v) for k, v in arrays.items()})


def main():
    R = op.ref()
    # --- assemble_step (solver.cpp:23-77) on two grids, with and without G
    for tag, dims, h, tau, eps in [("a", (6, 5, 4, 5), 0.2, 0.05, 1e-3),
                                   ("b", (5, 4, 3, 4), 1.0 / 7, 0.3, 1e-2)]:
        g = op.Grid.make(dims, h)
        u = cs.rand_field(dims, 11, ghosts="random")
        G = cs.rand_G(dims, 12)
        st, off, dg, ab = R.assemble_step(g, u, G, tau, eps, 2)
        assert st == 0
        st0, off0, dg0, ab0 = R.assemble_step(g, u, None, tau, eps, 2)
        assert st0 == 0
        # redblack_sor (solver.cpp:379-397) on the assembled system, rhs = guess = u
        st, us, it, res = R.redblack_sor(g, off, u, u, 1.4, 1e-11, 500, 2)
        assert st == 0
        save(f"assemble_sor_{tag}", dims=np.array(dims), h=h, tau=tau, eps=eps, u=u, G=G,
             off=off, diag=dg, abar=ab, off_noG=off0, diag_noG=dg0, abar_noG=ab0,
             omega=1.4, tol=1e-11, sor_u=us, sor_iters=it, sor_res=res)

    # --- face_coefficients (edge.cpp:73-99) + heat_smooth (preprocess.cpp:25-51)
    dims = (6, 5, 4, 5)
    g = op.Grid.make(dims, 0.25)
    img = cs.f32_image(dims, 21)
    st, I0s = R.heat_smooth(g, img, np.sqrt(2) * 0.25, 1, 1.85, 1e-10, 10000, 2)
    assert st == 0
    rows = cs.centers_overlapping(dims)
    st, th = R.local_threshold(g, img, rows, 0.5, 0.0)
    assert st == 0
    st, ITs = R.heat_smooth(g, th, np.sqrt(2) * 0.25, 2, 1.85, 1e-10, 10000, 2)
    assert st == 0
    st, Gf = R.face_coefficients(g, I0s, ITs, 50.0, 0.5, 0.5, 2)
    assert st == 0
    save("preprocess", dims=np.array(dims), h=0.25, image=img, rows=np.array(rows),
         I0s=I0s, threshold=th, ITs=ITs, G=Gf, K=50.0, delta=0.5, vartheta=0.5)

    # --- build_initial / local_rescale (seedinit.cpp:42-99)
    st, u0 = R.build_initial(g, rows, 1.0, 3.0, 0)
    assert st == 0
    st, u0l = R.build_initial(g, rows, 0.5, 2.5, 1)
    assert st == 0
    noisy = cs.rand_field(dims, 31)
    st, resc_row = R.local_rescale(g, noisy, rows, None)
    assert st == 0
    st, resc_r2 = R.local_rescale(g, noisy, rows, 2.2)
    assert st == 0
    save("seedinit", dims=np.array(dims), h=0.25, rows=np.array(rows), u0_peak=u0,
         u0_linear=u0l, noisy=noisy, rescale_rowradius=resc_row, rescale_r22=resc_r2)

    # --- segment (solver.cpp:405-441), reference semantics (absolute tol) and harness (rel tol)
    dims = (8, 7, 6, 6)
    h = 1.0 / 8
    g = op.Grid.make(dims, h)
    img = cs.f32_image(dims, 41, noise=0.05)
    rows = [(f, 3.5, 3.0, 2.5, 2.0) for f in range(6)]
    p = op.seg_params(tau=h, epsilon=1e-3, omega=1.4, sor_tol=1e-9, n_steps=3,
                      sigma=np.sqrt(2) * h, K=200.0, delta=0.5, vartheta=0.5, rescale_radius=3.0)
    st, useg, info = R.segment(g, img, rows, p, None, 2)
    assert st == 0
    p2 = op.seg_params(tau=h, epsilon=1e-3, omega=1.4, sor_rel_tol=1e-8, n_steps=3,
                       sigma=np.sqrt(2) * h, K=200.0, delta=0.5, vartheta=0.5, rescale_radius=3.0)
    st, useg2, info2 = R.segment(g, img, rows, p2, None, 3)
    assert st == 0
    save("segment", dims=np.array(dims), h=h, image=img, rows=np.array(rows), u=useg,
         iters=np.array([d["iterations"] for d in info["diags"]]),
         u_rel=useg2, iters_rel=np.array([d["iterations"] for d in info2["diags"]]),
         res_rel=np.array([d["residual"] for d in info2["diags"]]),
         tol_rel=np.array([d["tol"] for d in info2["diags"]]))

    # --- EOC rows (eoc.cpp:83-137): Table-1 verification of the G == 1 path
    st, e10 = R.eoc_row(10, 1.5, 1e-8, 10000, 2)
    assert st == 0
    st, e20 = R.eoc_row(20, 1.5, 1e-8, 10000, 2)
    assert st == 0
    save("eoc", e10=e10, e20=e20)

    # --- tracking (tracking.cpp): extract_mask -> label_components -> distance_centers
    #     -> backtrack_link -> prolong_and_merge -> track on a moving-cells scene
    dims = (24, 20, 10, 8)
    g = op.Grid.make(dims, 1.0)
    u = cs.track_scene(dims, 5)
    m = R.extract_mask(g, u, 0.5)
    lab, lpf = R.label_components(g, m)
    rec = R.distance_centers(g, lab, lpf)
    chains = R.backtrack_link(g, lab, lpf)
    pts = R.track(g, u, 0.5, 3, 5.0)
    starts = np.cumsum([0] + [len(c) for c in chains])
    save("track", dims=np.array(dims), u=u, level=0.5, window=3, radius=5.0, labels=lab, lpf=np.array(lpf),
         records=rec, chain_fl=np.array([x for c in chains for x in c]), chain_start=starts,
         points=np.array([p[:2] for p in pts]), points_xyz=np.array([p[2:] for p in pts]))


if __name__ == "__main__":
    main()
