"""Where the host time of an e2e step goes (cfg1 / cfg4 stores from bench.py):
per next_many(G) call, the C call (rfl_loader_next_many: replay hand-off,
staging pull launch, assembly launch) vs the Python wrapping of the G batches
vs the per-step D2H read of the result ids, over N steps.

usage: python scripts/e2e_probe.py [cfg4|cfg1] [G] [steps]
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_01949_b200 as R  # noqa: E402
from paper_2604_01949_b200 import _lib as L  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 400
W = bench.WORKLOADS[wl]
path = bench.ensure_store(wl, 0, 1, None)
ds = R.DeviceStore(R.StoreReader(path), 0, os.environ.get("RIFFLE_E2E_STAGING", "stream_pinned"))
stream = torch.cuda.current_stream()
cfg = R.LoaderConfig(**W["loader"], prefetch_depth=4)
epoch = 0


def mk(e):
    return R.BatchIterator(ds, cfg, e, output=W["out"]["output"], out_dtype=W["out"]["out_dtype"],
                           transform=W["out"]["transform"], out_slots=3, stream=stream, batches_per_launch=G)


it = mk(0)
host = torch.empty(W["loader"]["batch_rows"] * G, dtype=torch.int64).pin_memory()
arr = (L.rfl_batch * G)()
host_ptr, stream_h = host.data_ptr(), stream.cuda_stream
n = C.c_uint32()
t_c = t_wrap = t_d2h = 0.0
done = 0
for warm in (True, False):
    if not warm:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
    k = 0
    while k < (4 * G if warm else steps):
        a = time.perf_counter()
        rc = L.check(L.lib().rfl_loader_next_many(it._h, arr, G, C.byref(n)))
        if rc == L.END:  # next epoch (as open_epoch), inside the timed region like bench.py's e2e leg
            epoch += 1
            it.close()
            it = mk(epoch)
            continue
        b = time.perf_counter()
        bs = [it._wrap(arr[i]) for i in range(n.value)]
        c = time.perf_counter()
        for bb in bs:
            bb.ids_to_host(host_ptr, stream_h)
        d = time.perf_counter()
        if not warm:
            t_c += b - a
            t_wrap += c - b
            t_d2h += d - c
        k += n.value
    if not warm:
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        done = k
rows = done * W["loader"]["batch_rows"]
print({"workload": wl, "G": G, "steps": done, "wall_ms": wall * 1e3, "rows_per_s": rows / wall,
       "us_per_step": {"c_call": 1e6 * t_c / done, "wrap": 1e6 * t_wrap / done, "d2h": 1e6 * t_d2h / done,
                       "total": 1e6 * wall / done},
       "epochs": epoch + 1})
