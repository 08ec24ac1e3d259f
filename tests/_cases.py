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
