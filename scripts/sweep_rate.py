"""Device time per SOR sweep (red + black pass + finalize, graph loop) on a config's
coefficients, plus the event-timed per-pass split.  Env SSB_SNAKE / SSB_L2HINT select
the pass order / L2 policies (read once per process)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2111_11866_b200 as ss
import workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "config1"
wl = workloads.CONFIGS[cfg]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g, n_slabs=int(os.environ.get("SLABS", "1")))
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 5}), wl.u0)
if os.environ.get("SUBSURF_KERNEL"):
    s.set_kernel(os.environ["SUBSURF_KERNEL"])
st = torch.cuda.ExternalStream(s.stream)
s.fixed_sweeps(20)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 200
e0.record(st)
s.fixed_sweeps(N)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1)
s.set_profiling(True)
s.profile()
s.fixed_sweeps(20)
pr = s.profile()
if os.environ.get("CHECK_VS_TMA"):  # bitwise check of the selected kernel against the TMA two-pass
    s.set_profiling(False)
    s.set_u(wl.u0 if wl.u0 is not None else s.get_u())
    s.fixed_sweeps(7)
    a = s.get_u()
    s.set_kernel("tma")
    s.set_u(wl.u0 if wl.u0 is not None else a)
    s.fixed_sweeps(7)
    print("bitwise_equal_to_tma", bool(np.array_equal(a, s.get_u())))
print(json.dumps(dict(config=cfg, ran=s.sor_kernel(), slabs=int(os.environ.get("SLABS", "1")), kernel=os.environ.get("SUBSURF_KERNEL"), lib=os.environ.get("SUBSURF_B200_LIB"), snake=os.environ.get("SSB_SNAKE"), l2hint=os.environ.get("SSB_L2HINT"),
                      us_per_sweep=1e3 * ms / N,
                      red_us=1e3 * pr["red_ms"] / max(1, pr["red_n"]),
                      black_us=1e3 * pr["black_ms"] / max(1, pr["black_n"]))))
