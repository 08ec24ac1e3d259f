"""The timed step of bench.py alone, for an ncu launch list: prepare + warmup steps outside,
then K time steps between cudaProfilerStart/Stop, the SOR loop host-driven (loop mode 0: every
colour pass a launch of its own, so ncu lists each).  Run under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv
      --log-file X.csv python scripts/step_launch_list.py [config4] [K]
the per-kernel shares of the step are then comparable with bench.py's sor_share_of_step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2111_11866_b200 as ss
import workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "config4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.config4(1) if cfg == "config4" else workloads.CONFIGS[cfg]()
fixed = wl.notes.get("fixed_sweeps")
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.set_loop_mode(0)
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 3 + K}), wl.u0)
step = (lambda: s.step_fixed(fixed, diag=False)) if fixed else s.step_nodiag
for _ in range(3):
    step()
torch.cuda.synchronize()
n0 = ss.launch_count()
torch.cuda.profiler.start()
for _ in range(K):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches in the profiled steps:", ss.launch_count() - n0)
