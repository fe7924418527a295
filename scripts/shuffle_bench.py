"""Pre-shuffle throughput on a Tahoe-shaped (config 5) collection: CSR,
62,710 genes, ~2,000 nnz/cell, input chunk 64, block c=64, out chunk 4096 x 128.

Reports, for the single-GPU writer (rfl_run_shuffle): wall rows/s and GB/s of
CSR payload end to end (input preads + H2D + device gather/permute/pack + D2H +
output writes), and the device kernels' own GB/s.  The reference run_shuffle
(oracle/_ref, the unmodified C++) is timed on a bounded subset beside it.

    python scripts/shuffle_bench.py [--rows 262144] [--m 65536] [--ref-rows 20000]
"""
import argparse
import json
import os
import shutil
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01949_b200 as R  # noqa: E402


def payload_bytes(path):
    return sum(f.stat().st_size for f in (Path(path) / "shards").iterdir())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=524288)
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--c", type=int, default=64)
    ap.add_argument("--ref-rows", type=int, default=20000)
    ap.add_argument("--dir", default=os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    args = ap.parse_args()
    base = Path(args.dir)
    base.mkdir(parents=True, exist_ok=True)
    src = base / f"cfg5_{args.rows}"
    if not (src / "manifest.json").exists():
        t = time.time()
        R.synth_store(src, R.SynthConfig(args.rows, 62710, "csr", "f32", "u32", 2000 / 62710, 4, 64, 128))
        print(f"# synth {time.time() - t:.1f}s", file=sys.stderr)
    nbytes = payload_bytes(src)
    import torch
    torch.zeros(1, device="cuda")  # CUDA context up before the clock starts (a process-level one-time cost)
    out = base / "cfg5_out"
    shutil.rmtree(out, ignore_errors=True)
    plan = R.plan_shuffle(args.rows, args.c, args.m, 7)
    t0 = time.perf_counter()
    st = R.run_shuffle([src], plan, out, R.ShuffleOutputConfig(4096, 128))
    wall = time.perf_counter() - t0
    res = {"workload": f"cfg5-shaped: {args.rows} cells x 62710 genes, ~2000 nnz/cell f32, c={args.c}, "
                       f"m={args.m}, out chunk 4096 x 128", "rounds": st.rounds_executed,
           "payload_GB": nbytes / 1e9, "wall_s": wall, "rows_per_s": args.rows / wall,
           "GBps_end_to_end": nbytes / wall / 1e9, "gpu_kernel_ms": st.gpu_ms,
           "GBps_kernels_payload": nbytes / (st.gpu_ms / 1e3) / 1e9,
           "h2d_GB": st.h2d_bytes / 1e9, "d2h_GB": st.d2h_bytes / 1e9,
           "peak_resident_rows": st.peak_resident_rows}
    shutil.rmtree(out, ignore_errors=True)
    if args.ref_rows:
        from oracle.oracle import Ref
        sub = base / f"cfg5_ref_{args.ref_rows}"
        if not (sub / "manifest.json").exists():
            R.synth_store(sub, R.SynthConfig(args.ref_rows, 62710, "csr", "f32", "u32", 2000 / 62710, 4, 64, 128))
        rout = base / "cfg5_ref_out"
        shutil.rmtree(rout, ignore_errors=True)
        t0 = time.perf_counter()
        Ref.run_shuffle([sub], rout, args.c, min(args.m, args.ref_rows), 7, 4096, 128)
        rw = time.perf_counter() - t0
        res["reference_cpu"] = {"rows": args.ref_rows, "wall_s": rw, "rows_per_s": args.ref_rows / rw,
                                "GBps": payload_bytes(sub) / rw / 1e9, "cores": 1,
                                "kind": "reference (oracle/_ref run_shuffle, single-threaded by design)"}
        shutil.rmtree(rout, ignore_errors=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
