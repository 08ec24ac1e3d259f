"""Seeded test inputs shared by the golden-fixture generator and the tests."""
from __future__ import annotations

import numpy as np


def grid(dims, h):
    from oracle.oracle_py import Grid
    return Grid.make(dims, h)


def shape(dims):
    n1, n2, n3, n4 = dims
    return (n4 + 2, n3 + 2, n2 + 2, n1 + 2)


def rand_field(dims, seed, lo=0.0, hi=1.0, ghosts="random"):
    rng = np.random.default_rng(seed)
    f = rng.uniform(lo, hi, size=shape(dims))
    if ghosts == "zero":
        g = np.zeros_like(f)
        g[1:-1, 1:-1, 1:-1, 1:-1] = f[1:-1, 1:-1, 1:-1, 1:-1]
        f = g
    return f


def rand_G(dims, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.05, 1.0, size=shape(dims) + (8,))


def f32_image(dims, seed, noise=0.1):
    """Blob + noise, rounded to float32 like read_image4d (io.cpp:81-94); ghosts 0."""
    n1, n2, n3, n4 = dims
    rng = np.random.default_rng(seed)
    l, k, j, i = np.meshgrid(np.arange(n4), np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    c = np.array([n1, n2, n3, n4]) / 2.0
    d = np.sqrt(((i - c[0]) / n1) ** 2 + ((j - c[1]) / n2) ** 2 + ((k - c[2]) / n3) ** 2
                + ((l - c[3]) / n4) ** 2)
    img = (d < 0.3).astype(np.float64) + rng.normal(0, noise, size=d.shape)
    out = np.zeros(shape(dims))
    out[1:-1, 1:-1, 1:-1, 1:-1] = img.astype(np.float32).astype(np.float64)
    return out


def centers_overlapping(dims):
    """Rows in several frames, some overlapping (order matters), radii 1.5..3."""
    n1, n2, n3, n4 = dims
    rows = [
        (0, (n1 - 1) / 2, (n2 - 1) / 2, (n3 - 1) / 2, 2.5),
        (0, (n1 - 1) / 2 + 1.0, (n2 - 1) / 2, (n3 - 1) / 2, 2.0),
        (min(1, n4 - 1), 1.0, 1.0, 0.0, 1.5),
        (n4 - 1, n1 - 1.0, n2 - 1.0, n3 - 1.0, 3.0),
        (0, (n1 - 1) / 2 - 0.5, (n2 - 1) / 2 + 0.5, (n3 - 1) / 2, 1.7),
    ]
    return rows


def to_centers(rows):
    from oracle.oracle_py import Center
    return [Center(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4])) for r in rows]


def track_scene(dims, seed, n_cells=6, noise_specks=12):
    """Padded u field (ghosts 0) of cells moving through the frames, for the
    tracking pipeline (tracking.cpp): ellipsoids drifting linearly, one cell
    dividing half-way, one cell missing in one frame (a gap the tangent
    prolongation of prolong_and_merge can bridge), two cells touching only
    diagonally (26-connectivity), and isolated single-voxel specks."""
    n1, n2, n3, n4 = dims
    rng = np.random.default_rng(seed)
    z, y, x = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    u = np.zeros(shape(dims))
    p0 = rng.uniform([3, 3, 2], [n1 - 4, n2 - 4, n3 - 3], size=(n_cells, 3))
    vel = rng.uniform(-1.2, 1.2, size=(n_cells, 3)) * np.array([1, 1, 0.5])
    ax = rng.uniform([1.5, 1.5, 1.2], [3.0, 3.0, 2.0], size=(n_cells, 3))
    gap_cell, gap_frame = 1, n4 // 2
    for f in range(n4):
        vol = np.zeros((n3, n2, n1))
        for c in range(n_cells):
            if c == gap_cell and f == gap_frame:
                continue
            ctr = p0[c] + vel[c] * f
            parts = [ctr]
            if c == 0 and f >= n4 // 2:  # division: two daughters drifting apart
                off = np.array([1.0 + 0.8 * (f - n4 // 2), 0.0, 0.0])
                parts = [ctr - off, ctr + off]
            for q in parts:
                d = ((x - q[0]) / ax[c, 0]) ** 2 + ((y - q[1]) / ax[c, 1]) ** 2 + ((z - q[2]) / ax[c, 2]) ** 2
                vol = np.maximum(vol, np.clip(1.2 - 0.6 * d, 0.0, 1.0))
        # two single voxels touching only at a corner, and random specks
        vol[1, 1, 1] = vol[2, 2, 2] = 0.9
        for _ in range(noise_specks):
            vol[rng.integers(0, n3), rng.integers(0, n2), rng.integers(0, n1)] = rng.uniform(0.5, 1.0)
        u[f + 1, 1:-1, 1:-1, 1:-1] = vol
    return u


def random_mask(dims, seed, density):
    rng = np.random.default_rng(seed)
    n1, n2, n3, n4 = dims
    return (rng.random((n4, n3, n2, n1)) < density).astype(np.uint8)
