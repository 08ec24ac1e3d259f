"""One rank's share of BASELINE config 3 at N = 2 on one GPU: 512x512x128 x 32 frames
(1.07e9 doxels) -- prepare + two fixed-sweep steps, device memory in use after each phase.
(The rank of a 2-GPU job also holds two halo planes; this grid has ghost planes there.)"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2111_11866_b200 as ss
import workloads
t0 = time.time()
wl = workloads.config3(planes=(0, 33))
n1, n2, n3, _ = wl.dims
wl.dims = (n1, n2, n3, 32)
wl.image[-1] = 0.0
wl.u0[-1] = 0.0
g = ss.Grid.make(wl.dims, wl.h)
gen = time.time() - t0
free0, total = torch.cuda.mem_get_info()
out = {"dims": list(wl.dims), "gen_s": gen, "total_gb": total / 1e9, "free_before_gb": free0 / 1e9}
with ss.Session(g) as s:
    t1 = time.time()
    s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 2}), wl.u0)
    torch.cuda.synchronize()
    out["prepare_s"] = time.time() - t1
    out["used_after_prepare_gb"] = (free0 - torch.cuda.mem_get_info()[0]) / 1e9
    t2 = time.time()
    d = [s.step_fixed(5) for _ in range(2)]
    out["two_steps_s"] = time.time() - t2
    out["used_after_steps_gb"] = (free0 - torch.cuda.mem_get_info()[0]) / 1e9
    out["diags"] = d
print(json.dumps(out))
