"""Seconds per segment() time step (SURVEY 8(d)'s second metric), this repo on one
B200 vs the unmodified reference (oracle/_ref, std::thread workers = min(host
threads, n4)) on the host cores of the same box, same workload, same steps.
Both: steps 1..S after the same prepare; the reference's per-step wall times come
from its own segment() loop (ref_segment step_seconds)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2111_11866_b200 as ss
import workloads
from oracle import oracle_py as op

cfg = sys.argv[1]
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.CONFIGS[cfg]()
g = ss.Grid.make(wl.dims, wl.h)
p = ss.seg_params(**{**wl.params, "n_steps": S})
s = ss.Session(g)
t0 = time.perf_counter()
s.prepare(wl.image, wl.rows, p, wl.u0)
prep = time.perf_counter() - t0
ours, its = [], []
for _ in range(S):
    t0 = time.perf_counter()
    d = s.step()
    ours.append(time.perf_counter() - t0)
    its.append(d["iterations"])
u_gpu = s.get_u()
s.close()
res = {"workload": wl.name, "steps": S, "gpu_prepare_s": prep, "gpu_step_s": ours, "gpu_iterations": its}
if op.ref_available() and not os.environ.get("NO_REF"):
    R = op.ref()
    og = op.Grid.make(wl.dims, wl.h)
    workers = min(R.lib.ref_hardware_threads(), wl.dims[3])
    t0 = time.perf_counter()
    st, u_ref, info = R.segment(og, wl.image, wl.rows, op.seg_params(**{**wl.params, "n_steps": S}), wl.u0, workers)
    res.update({"ref_workers": workers, "ref_total_s": time.perf_counter() - t0, "ref_setup_s": info["times"][0],
                "ref_step_s": info["step_seconds"], "ref_iterations": [x["iterations"] for x in info["diags"]],
                "u_identical": bool(np.array_equal(u_gpu, u_ref))})
    res["speedup_per_step"] = float(np.mean(res["ref_step_s"]) / np.mean(ours))
print(json.dumps(res))
