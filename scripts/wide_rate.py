"""µs per SOR sweep on a synthetic grid of any shape (default the paper's 567-wide frames),
for the kernel selected by SUBSURF_KERNEL / SSB_TILE2D: fixed sweeps on a smoothed
random image with G == 1 coefficients at a random u."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2111_11866_b200 as ss

dims = tuple(int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (567, 64, 32, 16)))
h = 1.0 / 64
g = ss.Grid.make(dims, h)
rng = np.random.default_rng(5)
img = np.zeros(g.shape)
img[g.interior] = rng.random((dims[3], dims[2], dims[1], dims[0])).astype(np.float32)
rows = [(f, dims[0] / 2, dims[1] / 2, dims[2] / 2, 4.0) for f in range(dims[3])]
p = ss.seg_params(tau=h, epsilon=1e-3, omega=1.4, sor_rel_tol=1e-8, n_steps=3, sigma=0.0, K=100.0, delta=0.5,
                  vartheta=0.5, rescale_radius=6.0)
s = ss.Session(g)
if os.environ.get("SUBSURF_KERNEL"):
    s.set_kernel(os.environ["SUBSURF_KERNEL"])
s.prepare(img, rows, p)
st = torch.cuda.ExternalStream(s.stream)
s.fixed_sweeps(10)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.fixed_sweeps(100)
e1.record(st)
e1.synchronize()
n = int(np.prod(dims))
us = 1e3 * e0.elapsed_time(e1) / 100
print(json.dumps(dict(dims=dims, kernel=os.environ.get("SUBSURF_KERNEL"), tile2d=os.environ.get("SSB_TILE2D"),
                      us_per_sweep=us, tb_per_s_56B=n * 56 / (us * 1e-6) / 1e12)))
