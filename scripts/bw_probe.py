"""HBM bandwidth probe for the SOR pass's traffic mix: pure read, copy, and an
8:1 read:write stream (what one SOR colour pass moves), CUDA-event timed."""
import json
import torch

N = 1 << 30  # bytes per buffer
a = torch.empty(N // 8, dtype=torch.float64, device="cuda").uniform_()
b = torch.empty_like(a)
small = torch.empty(N // 64, dtype=torch.float64, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


out = {}
s = t(lambda: a.sum())
out["read_GBps"] = N / s / 1e9
s = t(lambda: b.copy_(a))
out["copy_GBps"] = 2 * N / s / 1e9
# 8:1 mix: read 8 GB-equivalents per 1 written: a (1 GiB) read + small (1/8 GiB) write
s = t(lambda: (torch.sum(a), small.copy_(a[: N // 64])))
out["mix_read_plus_small_GBps"] = (N + 2 * N // 8) / s / 1e9
print(json.dumps(out))
