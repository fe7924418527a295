"""Host->device copy ceiling on this box: pinned H2D bandwidth for one large
copy and for many 1 MB copies (the loader's per-block staging granularity)."""
import json
import time

import torch

out = {}
n = 256 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
torch.cuda.synchronize()
out["h2d_256MB_GBps"] = 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
for chunk in (1 << 20, 256 << 10):
    k = n // chunk
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        e0.record()
        for i in range(k):
            d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    out[f"h2d_{chunk >> 10}KB_chunks_GBps"] = n / (e0.elapsed_time(e1) / 1e3) / 1e9
    out[f"h2d_{chunk >> 10}KB_chunks_host_us_per_call"] = (time.perf_counter() - t0) / k * 1e6
print(json.dumps(out))
