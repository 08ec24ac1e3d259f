"""Time only the SOR colour passes on config 1 coefficients (fixed sweeps, profiling on)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2111_11866_b200 as ss
import workloads
wl = workloads.config1()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.set_kernel("ldg")  # prepare (heat solves) with the LDG pass: the TMA build may be an experiment
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 5}), wl.u0)
s.set_kernel(os.environ.get("SUBSURF_KERNEL", "tma"))
s.fixed_sweeps(10)
s.set_profiling(True)
s.profile()
s.fixed_sweeps(30)
pr = s.profile()
print(json.dumps(dict(lib=os.path.basename(os.environ.get("SUBSURF_B200_LIB", "default")),
                      red_us=1e3 * pr["red_ms"] / max(1, pr["red_n"]), black_us=1e3 * pr["black_ms"] / max(1, pr["black_n"]))))
