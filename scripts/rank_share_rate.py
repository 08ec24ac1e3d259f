"""One rank's share of BASELINE config 3 (512x512x128x64, t-slabs) at N = 8 / 4 / 2 GPUs, measured
on one B200 as a grid of its own (workloads.config3_slab(64 / N): the same rows, planes and nuclei):
device time per red+black sweep in the CUDA-graph loop of fixed-sweep solves (the compute each rank
does per sweep), and the strong-scaling efficiency of that compute relative to N = 2.  The halo
exchange per colour pass (one colour-packed boundary plane to each neighbour, overlapped with the
interior slices) is reported as bytes and as a time at a stated NVLink rate -- a model,
not a measurement (gpurun has one GPU).  rank_share_rate.py [N ...] -> JSON lines."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2111_11866_b200 as ss
import workloads

NVLINK_GBPS = 900.0  # per direction, B200 NVLink 5 (nominal)
out = []
for N in [int(a) for a in sys.argv[1:]] or [8, 4, 2]:
    n4 = 64 // N
    wl = workloads.config3_slab(n4)
    g = ss.Grid.make(wl.dims, wl.h)
    with ss.Session(g) as s:
        s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 5}), wl.u0)
        st = torch.cuda.ExternalStream(s.stream)
        s.fixed_sweeps(10)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 3 * 50
        e0.record(st)
        for _ in range(3):
            s.fixed_sweeps(50)
        e1.record(st)
        e1.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / K
    n1, n2, n3 = wl.dims[:3]
    plane_bytes = ((n1 + 3) // 2 + 1 & ~1) * (n2 + 2) * (n3 + 2) * 8  # one colour of one padded plane
    halo_us = 2 * plane_bytes / (NVLINK_GBPS * 1e9) * 1e6  # both neighbours, one direction each
    rec = dict(config="config3", ranks=N, frames_per_rank=n4, doxels_per_rank=n1 * n2 * n3 * n4,
               us_per_sweep=us, halo_bytes_per_pass=2 * plane_bytes, halo_us_per_pass_at_900GBps=halo_us,
               pass_us=us / 2, note="compute of one rank's slab measured on one B200; halo time modelled")
    out.append(rec)
    print(json.dumps(rec), flush=True)
base = next((r for r in out if r["ranks"] == 2), None)
if base:
    for r in out:
        print(json.dumps(dict(ranks=r["ranks"], compute_strong_eff_vs_2=base["us_per_sweep"] * 2 / (r["us_per_sweep"] * r["ranks"]))))
