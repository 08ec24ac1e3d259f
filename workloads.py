"""Seeded synthetic workloads of BASELINE.json's configs.

The reference measures no public dataset; these generators stand in for the
BASELINE configs with the stated shapes, sizes and value distributions.  Both
bench arms (this repo's CUDA path and the reference's CPU solver) consume the
identical arrays: the image is rounded to float32 like read_image4d
(io.cpp:81-94), u0 is built directly from the config's formula (ghosts 0), and
the centres table uses 0-based doxel coordinates (io.hpp:21-27).

Conventions: doxel centre x = (i - 0.5) h for 1-based i;
RNG numpy default_rng(1000 + config).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    dims: tuple            # (n1, n2, n3, n4)
    h: float
    image: np.ndarray      # padded (n4+2, n3+2, n2+2, n1+2) fp64 (f32-valued), ghosts 0
    u0: np.ndarray         # padded, ghosts 0
    rows: list             # centres table rows (frame, x, y, z, radius)
    params: dict           # ss_seg_params fields
    n_steps: int
    notes: dict = field(default_factory=dict)

    @property
    def n_interior(self) -> int:
        n1, n2, n3, n4 = self.dims
        return n1 * n2 * n3 * n4


def _padded(dims, interior: np.ndarray) -> np.ndarray:
    n1, n2, n3, n4 = dims
    out = np.zeros((n4 + 2, n3 + 2, n2 + 2, n1 + 2))
    out[1:-1, 1:-1, 1:-1, 1:-1] = interior
    return out


def _coords(dims, h):
    """Doxel-centre coordinates (x, y, z, t) as broadcastable arrays, axes (l, k, j, i)."""
    n1, n2, n3, n4 = dims
    x = ((np.arange(n1) + 0.5) * h)[None, None, None, :]
    y = ((np.arange(n2) + 0.5) * h)[None, None, :, None]
    z = ((np.arange(n3) + 0.5) * h)[None, :, None, None]
    t = ((np.arange(n4) + 0.5) * h)[:, None, None, None]
    return x, y, z, t


def _base_params(h, n_steps, **over):
    p = dict(tau=h, epsilon=1e-3, omega=1.4, sor_tol=1e-8, sor_rel_tol=1e-8, sor_max_iter=10000,
             n_steps=n_steps, rescale_each_step=1, sigma=np.sqrt(2.0) * h, smooth_steps=1,
             smooth_tol=1e-10, smooth_max_iter=10000, smooth_omega=1.85, lambda_=0.5,
             background=0.0, K=1000.0, delta=0.5, vartheta=0.5, init_v=1.0, init_R=10.0,
             init_profile=0, rescale_radius=12.0)
    p.update(over)
    return p


def _u0_seeds(dims, h, seeds):
    """u0 = max over seeds of 1/(|x - s|_4 / h + 1) (BASELINE config 0 formula)."""
    x, y, z, t = _coords(dims, h)
    u = None
    for s in seeds:
        d = np.sqrt((x - s[0]) ** 2 + (y - s[1]) ** 2 + (z - s[2]) ** 2 + (t - s[3]) ** 2)
        v = 1.0 / (d / h + 1.0)
        u = v if u is None else np.maximum(u, v)
    return _padded(dims, u)


def config0() -> Workload:
    """32^4 hypersphere, r = 0.3 at (0.5,)*4, N(0, 0.05^2) noise."""
    dims, h = (32, 32, 32, 32), 1.0 / 32
    rng = np.random.default_rng(1000)
    x, y, z, t = _coords(dims, h)
    d = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2 + (t - 0.5) ** 2)
    img = (d <= 0.3).astype(np.float64) + rng.normal(0.0, 0.05, size=d.shape)
    image = _padded(dims, img.astype(np.float32).astype(np.float64))
    # one centre row per frame that intersects the ball, at (15.5, 15.5, 15.5), radius 1 voxel
    rows = []
    for l in range(dims[3]):
        tc = (l + 0.5) * h
        if abs(tc - 0.5) < 0.3:
            rows.append((l, 15.5, 15.5, 15.5, 1.0))
    u0 = _u0_seeds(dims, h, [(0.5, 0.5, 0.5, 0.5)])
    return Workload("config0: 32^4 4D hypersphere", dims, h, image, u0, rows,
                    _base_params(h, 10, rescale_radius=12.0), 10,
                    notes=dict(noise=0.05, threshold_radius=1, rescale_radius=12))


def config1() -> Workload:
    """64^4, two moving Gaussian blobs (peak 1, radius 0.12), bg 0.1, N(0, 0.08^2),
    5% salt-and-pepper in blob 1's 0.10-0.12 shell; seeds at each blob's t=0 centre."""
    dims, h = (64, 64, 64, 64), 1.0 / 64
    rng = np.random.default_rng(1001)
    x, y, z, t = _coords(dims, h)
    T = t  # t in (0, 1)
    c1 = [0.3 + (0.5 - 0.3) * T, 0.3 + (0.4 - 0.3) * T, 0.5 + 0 * T]
    c2 = [0.7 + (0.6 - 0.7) * T, 0.7 + (0.6 - 0.7) * T, 0.5 + 0 * T]
    d1 = np.sqrt((x - c1[0]) ** 2 + (y - c1[1]) ** 2 + (z - c1[2]) ** 2)
    d2 = np.sqrt((x - c2[0]) ** 2 + (y - c2[1]) ** 2 + (z - c2[2]) ** 2)
    bg = 0.1
    g1 = np.where(d1 <= 0.12, (1 - bg) * np.exp(-0.5 * (d1 / 0.06) ** 2), 0.0)
    g2 = np.where(d2 <= 0.12, (1 - bg) * np.exp(-0.5 * (d2 / 0.06) ** 2), 0.0)
    img = bg + np.maximum(g1, g2) + rng.normal(0.0, 0.08, size=d1.shape)
    shell = (d1 >= 0.10) & (d1 <= 0.12)
    sp = shell & (rng.random(d1.shape) < 0.05)
    img = np.where(sp, rng.integers(0, 2, size=d1.shape).astype(np.float64), img)
    image = _padded(dims, img.astype(np.float32).astype(np.float64))
    t0 = 0.5 * h
    s1 = (0.3 + 0.2 * t0, 0.3 + 0.1 * t0, 0.5, t0)
    s2 = (0.7 - 0.1 * t0, 0.7 - 0.1 * t0, 0.5, t0)
    rows = [(0, s1[0] / h - 0.5, s1[1] / h - 0.5, s1[2] / h - 0.5, 1.0),
            (0, s2[0] / h - 0.5, s2[1] / h - 0.5, s2[2] / h - 0.5, 1.0)]
    u0 = _u0_seeds(dims, h, [s1, s2])
    return Workload("config1: 64^4 two moving blobs", dims, h, image, u0, rows,
                    _base_params(h, 20, rescale_radius=10.0), 20,
                    notes=dict(noise=0.08, salt_pepper=0.05, threshold_radius=1, rescale_radius=10))


def small(dims=(16, 12, 10, 8), seed=7) -> Workload:
    """Tiny smoke / test case with config-0 parameters."""
    n1, n2, n3, n4 = dims
    h = 1.0 / n1
    rng = np.random.default_rng(seed)
    x, y, z, t = _coords(dims, h)
    c = (n1 * h / 2, n2 * h / 2, n3 * h / 2, n4 * h / 2)
    d = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 + (t - c[3]) ** 2)
    img = (d <= 0.25).astype(np.float64) + rng.normal(0.0, 0.05, size=d.shape)
    image = _padded(dims, img.astype(np.float32).astype(np.float64))
    rows = [(l, c[0] / h - 0.5, c[1] / h - 0.5, c[2] / h - 0.5, 1.0) for l in range(n4)]
    u0 = _u0_seeds(dims, h, [c])
    return Workload(f"small {dims}", dims, h, image, u0, rows, _base_params(h, 3, rescale_radius=4.0), 3)


CONFIGS = {"config0": config0, "config1": config1}
