"""SOR loop on a config's coefficients for ~4 s with nvidia-smi sampled every 50 ms:
median SM clock and board power under load, and the us per sweep -- power_probe.py [config].
Variant libraries via SUBSURF_B200_LIB (scripts/build_variant.sh)."""
import json, os, subprocess, statistics, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2111_11866_b200 as ss
import workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "config4"
wl = workloads.CONFIGS[cfg]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 5}), wl.u0)
if os.environ.get("SUBSURF_KERNEL"):
    s.set_kernel(os.environ["SUBSURF_KERNEL"])
st = torch.cuda.ExternalStream(s.stream)
s.fixed_sweeps(20)
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks.mem", "--format=csv,noheader,nounits",
                         "-lms", "50", "-i", "0"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [lines.append(l) for l in proc.stdout], daemon=True)
th.start()
time.sleep(1.0)
lines.clear()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 3000 if wl.n_interior > 5e7 else 20000
e0.record(st)
s.fixed_sweeps(N)
e1.record(st)
e1.synchronize()
proc.terminate()
ms = e0.elapsed_time(e1)
vals = [[float(x) for x in l.split(",")] for l in lines if l.count(",") == 2]
vals = vals[len(vals) // 4:]  # steady state
print(json.dumps(dict(config=cfg, lib=os.environ.get("SUBSURF_B200_LIB"), kernel=os.environ.get("SUBSURF_KERNEL"), us_per_sweep=1e3 * ms / N,
                      sm_mhz=statistics.median(v[0] for v in vals), power_w=statistics.median(v[1] for v in vals),
                      mem_mhz=statistics.median(v[2] for v in vals), samples=len(vals))))
