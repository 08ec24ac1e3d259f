"""Event-timed SOR pass duration and step time for the library selected by
SUBSURF_B200_LIB (variant sweeps).  Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2111_11866_b200 as ss  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config1"
wl = workloads.CONFIGS[cfg]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.set_kernel(os.environ.get("SUBSURF_KERNEL", "tma"))
p = ss.seg_params(**{**wl.params, "n_steps": 10})
s.prepare(wl.image, wl.rows, p, wl.u0)
for _ in range(3):
    s.step_nodiag()
s.profile()
t0 = time.perf_counter()
for _ in range(3):
    s.step_nodiag()
dt = time.perf_counter() - t0
sweeps = s.profile()["sweeps"]
s.set_profiling(True)
s.step_nodiag()
pr = s.profile()
out = dict(lib=os.path.basename(os.environ.get("SUBSURF_B200_LIB", "default")), cfg=cfg,
           kernel=os.environ.get("SUBSURF_KERNEL", "tma"),
           red_us=1e3 * pr["red_ms"] / max(1, pr["red_n"]), black_us=1e3 * pr["black_ms"] / max(1, pr["black_n"]),
           sweep_us_wall=1e6 * dt / sweeps, assemble_us=1e3 * pr["assemble_ms"] / max(1, pr["assemble_n"]),
           value=wl.n_interior * sweeps / dt)
n = wl.n_interior
out["frac56"] = 28.0 * n / ((out["red_us"] + out["black_us"]) / 2 * 1e-6) / 6535.7e9
print(json.dumps(out))
