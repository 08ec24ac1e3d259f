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


def _config1_frames(frames, h, n_total):
    """Interior image planes of config 1 for the given 0-based global frames.

    Weak scaling repeats the 64-frame config along t (frame f uses the config-1
    time of frame f mod 64); the noise of every frame comes from its own seeded
    generator, so any rank can build exactly its slab."""
    n = 64
    x = ((np.arange(n) + 0.5) * h)[None, None, :]
    y = ((np.arange(n) + 0.5) * h)[None, :, None]
    z = ((np.arange(n) + 0.5) * h)[:, None, None]
    out = np.empty((len(frames), n, n, n))
    for q, f in enumerate(frames):
        rng = np.random.default_rng([1001, int(f)])
        T = ((f % 64) + 0.5) * h
        c1 = (0.3 + 0.2 * T, 0.3 + 0.1 * T, 0.5)
        c2 = (0.7 - 0.1 * T, 0.7 - 0.1 * T, 0.5)
        d1 = np.sqrt((x - c1[0]) ** 2 + (y - c1[1]) ** 2 + (z - c1[2]) ** 2)
        d2 = np.sqrt((x - c2[0]) ** 2 + (y - c2[1]) ** 2 + (z - c2[2]) ** 2)
        bg = 0.1
        g1 = np.where(d1 <= 0.12, (1 - bg) * np.exp(-0.5 * (d1 / 0.06) ** 2), 0.0)
        g2 = np.where(d2 <= 0.12, (1 - bg) * np.exp(-0.5 * (d2 / 0.06) ** 2), 0.0)
        img = bg + np.maximum(g1, g2) + rng.normal(0.0, 0.08, size=d1.shape)
        shell = (d1 >= 0.10) & (d1 <= 0.12)
        sp = shell & (rng.random(d1.shape) < 0.05)
        img = np.where(sp, rng.integers(0, 2, size=d1.shape).astype(np.float64), img)
        out[q] = img.astype(np.float32).astype(np.float64)
    return out


def config1(replicas: int = 1, planes=None) -> Workload:
    """64^4 (x replicas along t), two moving Gaussian blobs (peak 1, radius 0.12),
    bg 0.1, N(0, 0.08^2), 5% salt-and-pepper in blob 1's 0.10-0.12 shell; seeds at
    each blob's t=0 centre (of every 64-frame replica).

    planes=(p0, p1): build only padded planes p0..p1 (inclusive) of the global
    padded arrays -- a rank's slab plus halos -- instead of the whole grid."""
    n4 = 64 * replicas
    dims, h = (64, 64, 64, n4), 1.0 / 64
    p0, p1 = (0, n4 + 1) if planes is None else planes
    frames = [p - 1 for p in range(p0, p1 + 1)]
    inner = [f for f in frames if 0 <= f < n4]
    image = np.zeros((p1 - p0 + 1, 66, 66, 66))
    u0 = np.zeros_like(image)
    if inner:
        q0 = inner[0] - (p0 - 1)
        image[q0:q0 + len(inner), 1:-1, 1:-1, 1:-1] = _config1_frames(inner, h, n4)
    t0 = 0.5 * h
    s1 = (0.3 + 0.2 * t0, 0.3 + 0.1 * t0, 0.5)
    s2 = (0.7 - 0.1 * t0, 0.7 - 0.1 * t0, 0.5)
    x = ((np.arange(64) + 0.5) * h)[None, None, :]
    y = ((np.arange(64) + 0.5) * h)[None, :, None]
    z = ((np.arange(64) + 0.5) * h)[:, None, None]
    rows = []
    for r in range(replicas):
        rows.append((64 * r, s1[0] / h - 0.5, s1[1] / h - 0.5, s1[2] / h - 0.5, 1.0))
        rows.append((64 * r, s2[0] / h - 0.5, s2[1] / h - 0.5, s2[2] / h - 0.5, 1.0))
    for q, f in enumerate(frames):
        if not 0 <= f < n4:
            continue
        t = (f + 0.5) * h
        v = None
        for r in range(replicas):  # u0 = max over seeds of 1/(|x - s|_4 / h + 1)
            tr = 64 * r * h + t0
            for s in (s1, s2):
                d = np.sqrt((x - s[0]) ** 2 + (y - s[1]) ** 2 + (z - s[2]) ** 2 + (t - tr) ** 2)
                val = 1.0 / (d / h + 1.0)
                v = val if v is None else np.maximum(v, val)
        u0[q, 1:-1, 1:-1, 1:-1] = v
    name = "config1: 64^4 two moving blobs" + (f" x{replicas} along t (weak scaling)" if replicas > 1 else "")
    return Workload(name, dims, h, image, u0, rows, _base_params(h, 20, rescale_radius=10.0), 20,
                    notes=dict(noise=0.08, salt_pepper=0.05, threshold_radius=1, rescale_radius=10,
                               replicas=replicas, planes=(p0, p1)))


def _nuclei_tracks(n_nuclei, dims, n_frames, seed):
    """Seeded nucleus trajectories (config 2/3): start position, semi-axes U[4,8]
    voxels, intensity U[0.4,1], a N(0, 1.5^2)-per-frame random walk; 10% divide
    once into two daughters 6 voxels apart that walk on independently.
    Returns [(birth_frame, death_frame, positions[f] (x,y,z), axes, intensity)]."""
    n1, n2, n3 = dims
    rng = np.random.default_rng(seed)
    tracks = []
    for _ in range(n_nuclei):
        axes = rng.uniform(4.0, 8.0, size=3)
        inten = rng.uniform(0.4, 1.0)
        p = np.array([rng.uniform(8, n1 - 9), rng.uniform(8, n2 - 9), rng.uniform(6, n3 - 7)])
        divide_at = int(rng.integers(1, n_frames)) if rng.random() < 0.10 and n_frames > 1 else -1
        pos = np.zeros((n_frames, 3))
        for f in range(n_frames):
            pos[f] = p
            p = p + rng.normal(0.0, 1.5, size=3)
            p = np.clip(p, [2, 2, 2], [n1 - 3, n2 - 3, n3 - 3])
        if divide_at < 0:
            tracks.append((0, n_frames, pos, axes, inten))
            continue
        tracks.append((0, divide_at, pos, axes, inten))
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        for sgn in (-1.0, 1.0):
            q = pos[divide_at] + sgn * 3.0 * d
            dpos = pos.copy()
            for f in range(divide_at, n_frames):
                dpos[f] = q
                q = np.clip(q + rng.normal(0.0, 1.5, size=3), [2, 2, 2], [n1 - 3, n2 - 3, n3 - 3])
            tracks.append((divide_at, n_frames, dpos, axes * 0.8, inten))
    return tracks


def _nuclei_frame(dims, f, tracks, seed):
    """One frame (z, y, x) of the nuclei volume: background N(0.05, 0.03^2) blurred
    with a 2-voxel Gaussian, plus the ellipsoids alive in frame f (max-combined)."""
    from scipy.ndimage import gaussian_filter
    n1, n2, n3 = dims
    rng = np.random.default_rng([seed, int(f)])
    img = gaussian_filter(rng.normal(0.05, 0.03, size=(n3, n2, n1)).astype(np.float32), 2.0).astype(np.float64)
    for b, e, pos, axes, inten in tracks:
        if not b <= f < e:
            continue
        c = pos[f]
        lo = np.maximum(np.floor(c - axes).astype(int), 0)
        hi = np.minimum(np.ceil(c + axes).astype(int) + 1, [n1, n2, n3])
        x = np.arange(lo[0], hi[0])[None, None, :]
        y = np.arange(lo[1], hi[1])[None, :, None]
        z = np.arange(lo[2], hi[2])[:, None, None]
        inside = ((x - c[0]) / axes[0]) ** 2 + ((y - c[1]) / axes[1]) ** 2 + ((z - c[2]) / axes[2]) ** 2 <= 1.0
        sub = img[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        np.maximum(sub, np.where(inside, inten, 0.0), out=sub)
    return img.astype(np.float32).astype(np.float64)


def _nuclei_workload(name, dims, n_nuclei, seed, n_steps, planes, h=1.0 / 32, **over):
    n1, n2, n3, n4 = dims
    tracks = _nuclei_tracks(n_nuclei, (n1, n2, n3), n4, seed)
    p0, p1 = (0, n4 + 1) if planes is None else planes
    image = np.zeros((p1 - p0 + 1, n3 + 2, n2 + 2, n1 + 2))
    u0 = np.zeros_like(image)
    # one seed per nucleus at its first-frame centre; ball = the nucleus + 2 voxels
    rows = [(b, pos[b][0], pos[b][1], pos[b][2], float(axes.max()) + 2.0)
            for b, e, pos, axes, inten in tracks if b == 0]
    x = ((np.arange(n1) + 0.5) * h)[None, None, :]
    y = ((np.arange(n2) + 0.5) * h)[None, :, None]
    z = ((np.arange(n3) + 0.5) * h)[:, None, None]
    for q, p in enumerate(range(p0, p1 + 1)):
        f = p - 1
        if not 0 <= f < n4:
            continue
        image[q, 1:-1, 1:-1, 1:-1] = _nuclei_frame((n1, n2, n3), f, tracks, seed)
        if f == 0:  # u0: peak profile 1/(d/h + 1) around every seed of frame 0 (max-combined)
            v = np.zeros((n3, n2, n1))
            for r in rows:
                c = (np.array(r[1:4]) + 0.5) * h
                lo = np.maximum(np.floor(np.array(r[1:4]) - 12).astype(int), 0)
                hi = np.minimum(np.ceil(np.array(r[1:4]) + 13).astype(int), [n1, n2, n3])
                d = np.sqrt((x[..., lo[0]:hi[0]] - c[0]) ** 2 + (y[:, lo[1]:hi[1]] - c[1]) ** 2
                            + (z[lo[2]:hi[2]] - c[2]) ** 2)
                sub = v[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
                np.maximum(sub, 1.0 / (d / h + 1.0), out=sub)
            u0[q, 1:-1, 1:-1, 1:-1] = v
    params = _base_params(h, n_steps, K=5000.0, lambda_=0.7, rescale_radius=None, **over)
    return Workload(name, dims, h, image, u0, rows, params, n_steps,
                    notes=dict(nuclei=n_nuclei, h=h, threshold="0.3 -> lambda 0.7", planes=(p0, p1)))


def config2(planes=None) -> Workload:
    """256x256x64 x 32 frames, ~150 nuclei, K=5000, threshold 0.3, 30 steps (h = 1/32)."""
    return _nuclei_workload("config2: 256x256x64x32 nuclei", (256, 256, 64, 32), 150, 1002, 30, planes)


def config3(planes=None) -> Workload:
    """512x512x128 x 64 frames, ~2000 nuclei, 10 steps, omega 1.4 (>= 2 GPUs)."""
    return _nuclei_workload("config3: 512x512x128x64 nuclei", (512, 512, 128, 64), 2000, 1003, 10, planes)


def config3_slab(n4: int = 4) -> Workload:
    """The first n4 frames of config 3 (512x512x128, ~2000 nuclei) as a grid of their own:
    config 3's full-width rows and planes on one GPU (a parity case; the whole config 3
    needs >= 2 GPUs)."""
    wl = config3(planes=(0, n4 + 1))
    n1, n2, n3, _ = wl.dims
    wl.dims = (n1, n2, n3, n4)
    wl.image[-1] = 0.0  # the slab's upper ghost plane (the 64-frame grid's frame n4 + 1 otherwise)
    wl.u0[-1] = 0.0
    wl.rows = [r for r in wl.rows if r[0] < n4]
    wl.name = f"config3 slab: 512x512x128x{n4} (config 3's first {n4} frames)"
    return wl


def config4(gpus: int = 1, planes=None) -> Workload:
    """Weak scaling: 256x256x128 x (16 * gpus) frames, config-2 data and solver
    settings, fixed 50 SOR sweeps per time step (no early stop)."""
    wl = _nuclei_workload(f"config4: 256x256x128x{16 * gpus} nuclei (fixed 50 sweeps/step)",
                          (256, 256, 128, 16 * gpus), 150 * gpus, 1004, 2, planes)
    wl.notes["fixed_sweeps"] = 50
    return wl


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


def tiny(gpus: int = 1, planes=None) -> Workload:
    """A small weak-scaled grid (24x20x12 x 6 frames per GPU, config-0 parameters) for
    exercising bench.py's multi-rank path in tests; planes as in config1."""
    dims = (24, 20, 12, 6 * gpus)
    wl = small(dims, seed=17)
    wl.name = f"tiny: 24x20x12x{6 * gpus} ball (bench-path test)"
    if planes is not None:
        p0, p1 = planes
        wl.image = wl.image[p0:p1 + 1].copy()
        wl.u0 = wl.u0[p0:p1 + 1].copy()
    return wl


CONFIGS = {"config0": config0, "config1": config1, "config2": config2, "config3": config3,
           "config4": config4, "tiny": tiny}
