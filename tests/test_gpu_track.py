"""Cell tracking on the GPU (tracking.cpp) against the reference.

* golden fixture (tests/golden/track.npz, made by the unmodified reference): labels,
  cell records, backtrack chains and trajectory points, exact;
* the reference itself (oracle/_ref, prebuilt) on random masks and moving-cell scenes:
  labels, records, chains and points exact;
* Session.track on a device-resident segmentation == reference track() of the same u.
"""
import os

import numpy as np
import pytest

import _cases as cs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rec_rows(records):
    return np.array([[r.frame, r.label, r.cx, r.cy, r.cz, r.max_distance, r.voxel_count] for r in records],
                    dtype=np.int64).reshape(-1, 7)


def test_golden_track(gpu):
    d = np.load(os.path.join(GOLD, "track.npz"))
    dims = tuple(int(x) for x in d["dims"])
    g = gpu.Grid.make(dims, 1.0)
    m = gpu.extract_mask(d["u"], g, float(d["level"]))
    lab, lpf = gpu.label_components(m, g)
    assert lpf == d["lpf"].tolist()
    assert np.array_equal(lab, d["labels"])
    rec = gpu.distance_centers(lab, lpf, g)
    assert np.array_equal(rec_rows(rec), d["records"])
    chains = gpu.backtrack_link(rec, lab, lpf, g)
    fl = [(rec[i].frame, rec[i].label) for c in chains for i in c]
    assert fl == [tuple(x) for x in d["chain_fl"].tolist()]
    assert np.array_equal(np.cumsum([0] + [len(c) for c in chains]), d["chain_start"])
    pts = gpu.track(d["u"], g, float(d["level"]), int(d["window"]), float(d["radius"]))
    assert [p[:2] for p in pts] == [tuple(x) for x in d["points"].tolist()]
    assert np.array_equal(np.array([p[2:] for p in pts]), d["points_xyz"])


@pytest.mark.parametrize("dims,density,seed", [((9, 7, 5, 3), 0.3, 1), ((16, 12, 8, 2), 0.5, 2),
                                               ((33, 17, 5, 2), 0.65, 3), ((1, 1, 1, 2), 1.0, 4),
                                               ((40, 30, 20, 2), 0.08, 5)])
def test_labels_and_centers_random(gpu, ref, dims, density, seed):
    from oracle.oracle_py import Grid
    og = Grid.make(dims, 1.0)
    g = gpu.Grid.make(dims, 1.0)
    m = cs.random_mask(dims, seed, density)
    lab_r, lpf_r = ref.label_components(og, m)
    lab, lpf = gpu.label_components(m, g)
    assert lpf == lpf_r
    assert np.array_equal(lab, lab_r)
    rec = gpu.distance_centers(lab, lpf, g)
    assert np.array_equal(rec_rows(rec), ref.distance_centers(og, lab_r, lpf_r))


def test_empty_and_full_masks(gpu, ref):
    from oracle.oracle_py import Grid
    dims = (6, 5, 4, 3)
    g, og = gpu.Grid.make(dims, 1.0), Grid.make(dims, 1.0)
    for m in (np.zeros((3, 4, 5, 6), np.uint8), np.ones((3, 4, 5, 6), np.uint8)):
        lab, lpf = gpu.label_components(m, g)
        lab_r, lpf_r = ref.label_components(og, m)
        assert lpf == lpf_r and np.array_equal(lab, lab_r)
        rec = gpu.distance_centers(lab, lpf, g)
        assert np.array_equal(rec_rows(rec), ref.distance_centers(og, lab_r, lpf_r))
    u = np.zeros(g.shape)
    assert gpu.track(u, g) == ref.track(og, u)


@pytest.mark.parametrize("dims,seed,window,radius", [((24, 20, 10, 8), 7, 3, 5.0), ((32, 28, 12, 10), 8, 2, 3.0),
                                                     ((20, 20, 8, 12), 9, 4, 8.0)])
def test_track_scenes(gpu, ref, dims, seed, window, radius):
    from oracle.oracle_py import Grid
    og = Grid.make(dims, 1.0)
    g = gpu.Grid.make(dims, 1.0)
    u = cs.track_scene(dims, seed)
    m = gpu.extract_mask(u, g)
    lab, lpf = gpu.label_components(m, g)
    rec = gpu.distance_centers(lab, lpf, g)
    chains = gpu.backtrack_link(rec, lab, lpf, g)
    fl = [[(rec[i].frame, rec[i].label) for i in c] for c in chains]
    assert fl == ref.backtrack_link(og, lab, lpf)
    assert gpu.track(u, g, 0.5, window, radius) == ref.track(og, u, 0.5, window, radius)


def test_session_track_after_segment(gpu, ref):
    from oracle.oracle_py import Grid
    dims, h = (16, 12, 10, 6), 1.0 / 16
    g, og = gpu.Grid.make(dims, h), Grid.make(dims, h)
    img = cs.f32_image(dims, 77, noise=0.05)
    rows = [(f, 7.5, 5.5, 4.5, 2.0) for f in range(dims[3])]
    p = gpu.seg_params(tau=h, epsilon=1e-3, omega=1.4, sor_rel_tol=1e-8, n_steps=3, sigma=np.sqrt(2) * h,
                       K=200.0, delta=0.5, vartheta=0.5, rescale_radius=4.0)
    for slabs in (1, 3):
        s = gpu.Session(g, n_slabs=slabs)
        s.prepare(img, rows, p)
        for _ in range(3):
            s.step()
        u = s.get_u()
        got = s.track(0.5, 3, 5.0)
        s.close()
        assert got == ref.track(og, u, 0.5, 3, 5.0)
        assert len(got) > 0
