"""Tracking (tracking.cpp) on a config-2-sized field: the GPU
pipeline (Session.track on a device-resident u: labelling, distance transform,
centres, predecessor candidates on the GPU; linking on the host) vs the
reference's own track() (oracle/_ref, single-threaded CPU) on the same u.
u = the config-2 nuclei image (256x256x64 x 32 frames, ~150 nuclei), level 0.3."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2111_11866_b200 as ss
import workloads
from oracle import oracle_py as op

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
wl = workloads.CONFIGS[cfg]()
u = np.ascontiguousarray(wl.image)
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.set_u(u)
s.track(0.3, 3, 5.0)  # warm-up (allocations, module load)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    pts = s.track(0.3, 3, 5.0)
    ts.append(time.perf_counter() - t0)
res = {"workload": wl.name, "voxels": int(np.prod(wl.dims)), "points": len(pts),
       "trajectories": len({p[0] for p in pts}), "gpu_session_track_s": min(ts)}
t0 = time.perf_counter()
pts1 = ss.track(u, g, 0.3, 3, 5.0)
res["gpu_track_with_h2d_s"] = time.perf_counter() - t0
if op.ref_available() and "--no-ref" not in sys.argv:
    t0 = time.perf_counter()
    want = op.ref().track(op.Grid.make(wl.dims, wl.h), u, 0.3, 3, 5.0)
    res["reference_track_s"] = time.perf_counter() - t0
    res["identical_to_reference"] = want == pts and want == pts1
    res["speedup_session_vs_reference"] = res["reference_track_s"] / res["gpu_session_track_s"]
print(json.dumps(res))
