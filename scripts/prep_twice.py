"""prepare() twice in one process (the second is warm), wall times per phase (SSB_TIMING)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2111_11866_b200 as ss
import workloads
wl = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config1"]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
p = ss.seg_params(**{**wl.params, "n_steps": 2})
for k in range(2):
    t0 = time.perf_counter()
    s.prepare(wl.image, wl.rows, p, wl.u0)
    print(f"prepare #{k + 1}: {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
u = np.empty(g.shape)
for k in range(2):
    t0 = time.perf_counter()
    s.get_u_ptr(u.ctypes.data) if hasattr(s, "get_u_ptr") else s.get_u()
    print(f"get_u #{k + 1}: {time.perf_counter() - t0:.4f} s", file=sys.stderr, flush=True)
for k in range(2):
    t0 = time.perf_counter()
    s.set_u_ptr(u.ctypes.data)
    print(f"set_u #{k + 1}: {time.perf_counter() - t0:.4f} s", file=sys.stderr, flush=True)
