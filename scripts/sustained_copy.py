"""Sustained HBM copy under the board's power cap: torch b.copy_(a) (1 GiB each) back to back
for ~5 s with nvidia-smi sampled every 50 ms; read+write bytes / time, median SM clock and
power of the steady state.  The number a long-running bandwidth-bound step can expect, next to
MEASURED_PEAKS.json's burst copy (best of 10 short copies)."""
import json, statistics, subprocess, threading, time
import torch

N = 1 << 30
a = torch.empty(N // 8, dtype=torch.float64, device="cuda").uniform_()
b = torch.empty_like(a)
for _ in range(5):
    b.copy_(a)
torch.cuda.synchronize()
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                         "-lms", "50", "-i", "0"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [lines.append(l) for l in proc.stdout], daemon=True)
th.start()
time.sleep(1.0)
lines.clear()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
R = 2000
e0.record()
for _ in range(R):
    b.copy_(a)
e1.record()
e1.synchronize()
proc.terminate()
ms = e0.elapsed_time(e1)
vals = [[float(x) for x in l.split(",")] for l in lines if l.count(",") == 1]
vals = vals[len(vals) // 4:]
# burst: best of 10 single copies right after
best = 1e9
for _ in range(10):
    e0.record(); b.copy_(a); e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps(dict(sustained_copy_GBps=2 * N * R / (ms * 1e-3) / 1e9, seconds=ms / 1e3,
                      sm_mhz=statistics.median(v[0] for v in vals), power_w=statistics.median(v[1] for v in vals),
                      burst_copy_GBps_after=2 * N / (best * 1e-3) / 1e9, samples=len(vals))))
