"""Profiling driver: prepare BASELINE config (default config1) and run time steps.

Used under ncu on the GPU box (see profiles/README.md):
    python scripts/prof_step.py [--config config1] [--steps 2] [--loop-mode 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2111_11866_b200 as ss  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config1")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--loop-mode", type=int, default=0)
a = ap.parse_args()
wl = workloads.CONFIGS[a.config]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.set_loop_mode(a.loop_mode)
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": a.steps}), wl.u0)
for n in range(a.steps):
    d = s.step()
    print(f"step {n + 1}/{a.steps} sor_iters={d['iterations']} residual={d['residual']:.3e} "
          f"tol={d['tol']:.3e} min={d['umin']:.4f} max={d['umax']:.4f}")
s.close()
