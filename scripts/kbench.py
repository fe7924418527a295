"""Kernel micro-benchmark: every hot-path kernel on BASELINE-shaped synthetic
stores, device-resident, CUDA-event timed (K launches over K different row
sets, so nothing is served from L2), reported against the measured HBM peak.

    python scripts/kbench.py [--cases densify_cfg1,gather_cfg1,...] [--steps K]
Prints one JSON object per case.  Product code only (no oracle).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01949_b200 as R  # noqa: E402
from paper_2604_01949_b200 import _lib as L  # noqa: E402

STORES = {
    "cfg1": dict(n_obs=100_000, n_var=20_000, layout="csr", value_dtype="f32", density=0.1, seed=0, chunk_rows=64),
    "cfg2s": dict(n_obs=200_000, n_var=36_000, layout="csr", value_dtype="f32", density=3000 / 36000, seed=1,
                  chunk_rows=1024),
    "cfg3s": dict(n_obs=200_000, n_var=12288, layout="dense", value_dtype="u8", seed=2, chunk_rows=256),
    "cfg4s": dict(n_obs=1_000_000, n_var=4096, layout="dense", value_dtype="u8", seed=3, chunk_rows=512),
    "cfg4oh": dict(n_obs=1_000_000, n_var=4096, layout="dense", value_dtype="u8", seed=3, chunk_rows=512, one_hot=4),
    "cfg5s": dict(n_obs=65_536, n_var=62_710, layout="csr", value_dtype="f32", density=2000 / 62710, seed=4,
                  chunk_rows=64),
}
FULL_ROWS = {"cfg3s": 2_000_000, "cfg4s": 5_000_000}  # KB_FULL=1: BASELINE row counts (24.6 / 20.5 GB)
CASES = {  # store, kernel, rows per launch, out dtype, transform
    "densify_cfg1": ("cfg1", "densify", 4096, L.F32, L.XF_NONE),
    "densify_bf16_cfg1": ("cfg1", "densify", 4096, L.BF16, L.XF_NONE),
    "gather_cfg1": ("cfg1", "gather", 4096, None, None),
    "gather_planned_cfg1": ("cfg1", "gather_planned", 4096, None, None),
    "densify_norm_cfg2": ("cfg2s", "densify", 4096, L.F32, L.XF_NORMALIZE_LOG1P),
    "dense_bf16_cfg3": ("cfg3s", "dense", 1024, L.BF16, None),
    "dense_raw_cfg4": ("cfg4s", "dense", 2048, L.NATIVE, None),
    "dense_bf16_cfg3_g2": ("cfg3s", "dense", 2048, L.BF16, None),   # bench.py's 2 batches per launch
    "dense_raw_cfg4_g4": ("cfg4s", "dense", 8192, L.NATIVE, None),  # bench.py's 4 batches per launch
    "pack_cfg5": ("cfg5s", "pack", 65536, None, None),
    # K4o: one-hot rows from the HBM-resident 2-bit code image (resident_coded), as bench.py's value leg
    "onehot_cfg4": ("cfg4oh", "onehot", 2048, L.NATIVE, None),
    "onehot_cfg4_g10": ("cfg4oh", "onehot", 20480, L.NATIVE, None),
    "onehot_bf16_cfg4_g4": ("cfg4oh", "onehot", 8192, L.BF16, None),
}


GRAPH = False


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def store(name):
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    full = os.environ.get("KB_FULL") and name in FULL_ROWS  # the BASELINE-sized dense stores
    path = base / (f"kb_{name}_full" if full else f"kb_{name}")
    if not (path / "manifest.json").exists():
        base.mkdir(parents=True, exist_ok=True)
        t = time.time()
        s = dict(STORES[name])
        if full:
            s["n_obs"] = FULL_ROWS[name]
        R.synth_store(path, R.SynthConfig(**s))
        print(f"# synth {name}: {time.time() - t:.1f}s", file=sys.stderr)
    return path


def row_nnz(reader, man):
    out = np.zeros(man.n_obs, np.int64)
    for q in range(man.chunk_count()):
        rec = reader.read_record(q)
        rows = int(np.frombuffer(rec, np.uint32, 1, 0)[0])
        ip = np.frombuffer(rec, np.uint32, rows + 1, 12).astype(np.int64)
        out[q * man.chunk_rows:q * man.chunk_rows + rows] = np.diff(ip)
    return out


def run_case(name, K, W, dstores):
    import torch
    st_name, kern, rows, od, xf = CASES[name]
    if st_name not in dstores:
        dstores[st_name] = R.DeviceStore(store(st_name), 0, "resident_coded" if kern == "onehot" else "resident")
    ds = dstores[st_name]
    man = ds.manifest()
    base, offs = ds.arena()
    desc = ds.arena_desc()
    rng = np.random.default_rng(0)
    sets = [rng.choice(man.n_obs, rows, replace=False).astype(np.uint64) for _ in range(K + W)]
    if os.environ.get("KB_SCHED"):  # row sets = consecutive batches of the loader's own schedule
        f = man.chunk_rows
        it = iter(R.EpochSchedule(man.n_obs, R.LoaderConfig(f, max(16384, rows), rows, 0), 0))
        sets = [next(it).astype(np.uint64) for _ in range(K + W)]
    refs = np.zeros((K + W, rows, 2), np.uint64)
    for i, g in enumerate(sets):
        refs[i, :, 0] = offs[g.astype(np.int64) // man.chunk_rows]
        refs[i, :, 1] = g
    d_refs = torch.from_numpy(refs.view(np.int64)).cuda()
    lib = L.lib()
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    vs = {"f32": 4, "f64": 8, "i32": 4, "u8": 1}[man.value_dtype]
    isz = 4
    nnz = None
    if man.layout == "csr":
        rn = row_nnz(ds.reader, man)
        nnz = [int(rn[g.astype(np.int64)].sum()) for g in sets]
    gout = torch.empty(rows, dtype=torch.int64, device="cuda")
    def rotating(nbytes):  # output buffers totalling > 2 x L2: no launch writes over cached output
        n_out = max(2, -(-(256 << 20) // nbytes))
        return [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(n_out)]
    if kern == "densify":
        osz = 2 if od == L.BF16 else 4
        outs = rotating(rows * man.n_var * osz + 16)
        launch = lambda i: lib.rfl_csr_densify(C.byref(desc), d_refs[i].data_ptr(), rows, od, xf, 1e4,  # noqa
                                               outs[i % len(outs)].data_ptr(), gout.data_ptr(), sp)
        alg = lambda i: nnz[i] * (isz + vs) + rows * (16 + 2 * isz + man.n_var * osz + 8)  # noqa
    elif kern == "gather":
        mx = max(nnz)
        o_ip = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
        o_ix = torch.empty(mx * isz + 16, dtype=torch.uint8, device="cuda")
        o_dv = torch.empty(mx * vs + 16, dtype=torch.uint8, device="cuda")
        launch = lambda i: lib.rfl_csr_gather(C.byref(desc), d_refs[i].data_ptr(), rows, o_ip.data_ptr(),  # noqa
                                              o_ix.data_ptr(), o_dv.data_ptr(), gout.data_ptr(), sp)
        alg = lambda i: nnz[i] * 2 * (isz + vs) + rows * (16 + 2 * isz + 16)  # noqa
    elif kern == "gather_planned":  # indptr planned on the host (the loader's CSR path): one launch
        mx = max(nnz)
        pre = np.zeros((K + W, rows + 1), np.int64)
        for i, g in enumerate(sets):
            pre[i, 1:] = np.cumsum(rn[g.astype(np.int64)])
        d_pre = torch.from_numpy(pre).cuda()
        o_ix = torch.empty(mx * isz + 16, dtype=torch.uint8, device="cuda")
        o_dv = torch.empty(mx * vs + 16, dtype=torch.uint8, device="cuda")
        launch = lambda i: lib.rfl_csr_gather_prefixed(C.byref(desc), d_refs[i].data_ptr(), rows,  # noqa
                                                       d_pre[i].data_ptr(), o_ix.data_ptr(), o_dv.data_ptr(),
                                                       gout.data_ptr(), sp)
        alg = lambda i: nnz[i] * 2 * (isz + vs) + rows * (16 + 2 * isz + 16)  # noqa
    elif kern == "dense":
        rb = man.n_var * vs
        osz = 2 if od == L.BF16 else vs
        outs = rotating(rows * man.n_var * osz + 16)
        launch = lambda i: lib.rfl_dense_gather(C.byref(desc), d_refs[i].data_ptr(), rows, od,  # noqa
                                                outs[i % len(outs)].data_ptr(), gout.data_ptr(), sp)
        alg = lambda i: rows * (16 + rb + man.n_var * osz + 8)  # noqa
    elif kern == "onehot":
        osz = 2 if od == L.BF16 else 1
        outs = rotating(rows * man.n_var * osz + 16)
        launch = lambda i: lib.rfl_onehot_gather(C.byref(desc), d_refs[i].data_ptr(), rows, od,  # noqa
                                                 outs[i % len(outs)].data_ptr(), gout.data_ptr(), sp)
        alg = lambda i: rows * (16 + man.n_var // 16 + man.n_var * osz + 8)  # noqa
    else:  # pack: scan + record pack, 4096-row output chunks
        cr = 4096
        P = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
        mx = max(nnz)
        out = torch.empty(mx * (isz + vs) + (rows // cr + 1) * (12 + 4 * (cr + 1)) + 16, dtype=torch.uint8,
                          device="cuda")

        def launch(i):
            rc = lib.rfl_csr_scan(C.byref(desc), d_refs[i].data_ptr(), rows, P.data_ptr(), sp)
            if rc:
                return rc
            return lib.rfl_csr_pack(C.byref(desc), d_refs[i].data_ptr(), rows, cr, L.IDX_U32, P.data_ptr(),
                                    out.data_ptr(), sp)
        nch = (rows + cr - 1) // cr
        alg = lambda i: nnz[i] * 2 * (isz + vs) + rows * 2 * (16 + 2 * isz) + 12 * nch + 4 * (rows + nch)  # noqa
    for i in range(W):
        L.check(launch(i))
    torch.cuda.synchronize()
    if GRAPH:  # the K launches captured once, replayed back to back: device time without host launch gaps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            cs = torch.cuda.current_stream()
            sp.value = cs.cuda_stream
            for k in range(K):
                L.check(launch(W + k))
        sp.value = stream.cuda_stream
        g.replay()
        torch.cuda.synchronize()
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        g.replay()
        e0.record(stream)
        torch.cuda.synchronize()
        ms = [s0.elapsed_time(e0) / K] * K
    else:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            ev[k][0].record(stream)
            L.check(launch(W + k))
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        ms = [s.elapsed_time(e) for s, e in ev]
    a = [alg(W + k) for k in range(K)]
    gbs = sum(a) / (sum(ms) / 1e3) / 1e9
    return {"case": name, "kernel": kern, "graph": GRAPH, "rows_per_launch": rows, "ms_mean": float(np.mean(ms)),
            "ms_min": float(np.min(ms)), "alg_MB_per_launch": float(np.mean(a)) / 1e6, "GBps": gbs,
            "frac_of_measured_hbm": gbs / peak(), "rows_per_s": rows / (np.mean(ms) / 1e3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--graph", action="store_true", help="replay the K launches as one CUDA graph")
    args = ap.parse_args()
    global GRAPH
    GRAPH = args.graph
    dstores = {}
    for c in args.cases.split(","):
        print(json.dumps(run_case(c, args.steps, args.warmup, dstores)), flush=True)


if __name__ == "__main__":
    main()
