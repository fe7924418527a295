"""Where the end-to-end loader step goes: host time inside BatchIterator.next(),
device time per step, staged bytes, for one bench workload (stream_pinned)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_01949_b200 as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W = bench.WORKLOADS[wl]
path = bench.ensure_store(wl, 0, 1, None)
t = time.perf_counter()
ds = R.DeviceStore(R.StoreReader(path), 0, sys.argv[3] if len(sys.argv) > 3 else "stream_pinned")
t_ds = time.perf_counter() - t
stream = torch.cuda.current_stream()
it = R.BatchIterator(ds, R.LoaderConfig(**W["loader"], prefetch_depth=4), 0, output=W["out"]["output"],
                     out_dtype=W["out"]["out_dtype"], transform=W["out"]["transform"], out_slots=3, stream=stream)
host = torch.empty(W["loader"]["batch_rows"], dtype=torch.int64).pin_memory()
rows = []
for k in range(steps):
    t0 = time.perf_counter()
    b = it.next()
    t1 = time.perf_counter()
    host[:b.n_rows].copy_(b.global_indices, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    c = it.counters()
    rows.append({"step": k, "next_ms": (t1 - t0) * 1e3, "sync_ms": (t2 - t1) * 1e3, "h2d_MB": c.h2d_bytes / 1e6,
                 "blocks": c.blocks_fetched})
print(json.dumps({"workload": wl, "dstore_s": t_ds, "steps": rows}))
