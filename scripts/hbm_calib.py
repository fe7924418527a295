"""HBM calibration on this GPU: copy (read+write), write-only (memset / fill),
read-only (sum) bandwidth at the sizes the loader kernels move, CUDA-event timed.
Tells how far a write-dominated kernel (densify: ~83 % writes) can go."""
import json

import torch


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


out = {}
for mb in (64, 328, 1024):
    n = mb * 2**20
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    f = a.view(torch.float32)
    out[f"copy_{mb}MB_GBps"] = 2 * n / t(lambda: b.copy_(a)) / 1e9
    out[f"memset_{mb}MB_GBps"] = n / t(lambda: a.zero_()) / 1e9
    out[f"fill_{mb}MB_GBps"] = n / t(lambda: f.fill_(1.5)) / 1e9
    out[f"read_sum_{mb}MB_GBps"] = n / t(lambda: f.sum()) / 1e9
print(json.dumps(out))
