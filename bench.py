"""Benchmark: cells/sec minibatch assembly on B200 (BASELINE.json metric).

A *step* is the assembly of one minibatch (b rows) of the loader's epoch
stream.  Default workload = BASELINE config 1 (the single-GPU config; config 2
does not fit one GPU's HBM): synthetic CSR
100k cells x 20k genes, ~2k nnz/cell f32, f=64 rows/fetch, B=4096, b=4096,
densify to fp32.

  value  — device-resident: the store's chunk records resident in HBM and the
           step's row references precomputed on the device; K timed launches
           of the densify kernel.  Whole-job cells/s = N * cells / max-rank time.
  e2e    — the same metric through the public API (BatchIterator.next()) with
           the store in pinned host memory (re-encoded at open with u8 column
           deltas / u16 ids, lossless): every step stages the fetched blocks
           host->device (cudaMemcpyAsync), expands them on the GPU, replays the
           schedule on the host, assembles, and reads the batch's
           global_indices back.

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
        [--workload cfg1|cfg2|cfg3|cfg4]; N>1 under torchrun (one rank/GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: synth config, loader config, output
    "cfg1": dict(desc="cfg1: synthetic CSR 100k cells x 20k genes, ~2k nnz/cell f32 (density 0.1), chunk 64, "
                      "f=64 B=4096 b=4096, densify fp32",
                 synth=dict(n_obs=100_000, n_var=20_000, layout="csr", value_dtype="f32", index_dtype="u32",
                            density=0.1, seed=0, chunk_rows=64, chunks_per_shard=128),
                 loader=dict(fetch_block_rows=64, buffer_capacity_rows=4096, batch_rows=4096, seed=0),
                 out=dict(output="dense", out_dtype="f32", transform=None), dtype="f32"),
    "cfg2": dict(desc="cfg2: synthetic counts CSR 10M cells x 36k genes, 2k-4k nnz/cell (~3k; procedural, "
                      "SURVEY 8d), values 1..64 as f32, f=1024 B=16384 b=4096, densify fp32 + library-size/log1p",
                 synth=dict(n_obs=10_000_000, n_var=36_000, layout="csr", value_dtype="f32", index_dtype="u32",
                            density=3000 / 36000, seed=1, chunk_rows=1024, chunks_per_shard=128, counts=True),
                 # 240 GB of records: more than this box's disk (80 GB free) or RAM (196 GB), so the
                 # store is a procedural record source (byte-identical to synth_store's files,
                 # tests/test_host.py) and the device holds its re-encoded staging image (~70 GB)
                 procedural=True,
                 loader=dict(fetch_block_rows=1024, buffer_capacity_rows=16384, batch_rows=4096, seed=0),
                 out=dict(output="dense", out_dtype="f32", transform="normalize_log1p"), dtype="f32"),
    "cfg3": dict(desc="cfg3: dense 3x64x64 u8 crops (2M samples), chunk 256, f=256 B=16384 b=1024, cast bf16",
                 synth=dict(n_obs=2_000_000, n_var=12288, layout="dense", value_dtype="u8", density=0.1, seed=2,
                            chunk_rows=256, chunks_per_shard=128),
                 loader=dict(fetch_block_rows=256, buffer_capacity_rows=16384, batch_rows=1024, seed=0),
                 out=dict(output="dense", out_dtype="bf16", transform=None), dtype="u8->bf16", group=4, e2e_group=4,
                 e2e_min_steps=200),
    "cfg4": dict(desc="cfg4: dense 4x1024 one-hot u8 windows (5M, procedural one-hot: one channel per position), "
                      "chunk 512, f=512 B=16384 b=2048, raw u8",
                 synth=dict(n_obs=5_000_000, n_var=4096, layout="dense", value_dtype="u8", density=0.1, seed=3,
                            chunk_rows=512, chunks_per_shard=128, one_hot=4),
                 loader=dict(fetch_block_rows=512, buffer_capacity_rows=16384, batch_rows=2048, seed=0),
                 out=dict(output="dense", out_dtype="native", transform=None), dtype="u8", group=10, e2e_group=8,
                 e2e_min_steps=800,
                 # the value leg reads the rows from the store's HBM-resident coded image (2-bit channel
                 # codes, 1/16 of the records) like cfg2's: K4o writes each one-hot row from its codes
                 value_staging="resident_coded"),
}
METRIC = "cells/sec minibatch assembly"
# config 5 (pre-shuffle) at the largest shape that is materialised per run: CSR with the
# Tahoe gene count, ~2,000 nnz/cell, c=64, m=65,536 rows per round, out chunk 4096 x 128
CFG5 = dict(desc="cfg5-shaped pre-shuffle: synthetic CSR 524,288 cells x 62,710 genes, ~2k nnz/cell f32, c=64, "
                 "m=65,536 (8 rounds), plan seed 7, out chunk_rows 4096 x 128 per shard, codec none",
            synth=dict(n_obs=524_288, n_var=62_710, layout="csr", value_dtype="f32", index_dtype="u32",
                       density=2000 / 62_710, seed=4, chunk_rows=64, chunks_per_shard=128),
            c=64, m=65_536, seed=7, out_chunk_rows=4096, out_cps=128, ref_rows=20_000)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx: int):
        self.idx = idx
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def allreduce_max(x: float, dist) -> float:
    """Max over ranks (device tensor under NCCL, host tensor under gloo)."""
    if not dist:
        return float(x)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ensure_store(wl, rank, world, dist):
    import paper_2604_01949_b200 as R
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    path = base / wl
    s = (CFG5 if wl == "cfg5" else WORKLOADS[wl])["synth"]
    if rank == 0 and not (path / "manifest.json").exists():
        base.mkdir(parents=True, exist_ok=True)
        tmp = base / f".{wl}.{os.getpid()}"
        R.synth_store(tmp, R.SynthConfig(**s))
        os.replace(tmp, path)
    if dist:
        dist.barrier()
    return path


def schedule_batches(n_obs, lcfg, rank, world, need):
    """The exact global_indices stream of this rank, chained over epochs."""
    import paper_2604_01949_b200 as R
    out, epoch = [], 0
    while len(out) < need:
        cfg = R.LoaderConfig(**lcfg, rank=rank, world=world)
        for g in R.EpochSchedule(n_obs, cfg, epoch):
            out.append(g)
            if len(out) >= need:
                break
        epoch += 1
    return out


def procedural_spec(W):
    s = dict(W["synth"])
    if os.environ.get("RIFFLE_PROC_ROWS"):  # smaller runs of the same shape (diagnostics)
        s["n_obs"] = int(os.environ["RIFFLE_PROC_ROWS"])
    return (f"procedural:counts?n_obs={s['n_obs']}&n_var={s['n_var']}&seed={s['seed']}&chunk_rows={s['chunk_rows']}"
            f"&chunks_per_shard={s['chunks_per_shard']}&value_dtype={s['value_dtype']}")


def preshuffle_exchange_leg(rank, world, local, dist):
    """N > 1 only: a short multi-GPU pre-shuffle of a config-5-shaped collection
    (65,536 cells x 62,710 genes, ~2k nnz/cell, ~1 GB; c=64, m=16,384 -> 4 rounds;
    out chunk 4,096 rows x 2 per shard -> 8 shards, shard s owned by rank s mod W),
    through the public run_shuffle (exchange mode auto: fused peer stores when every
    GPU pair is peer-accessible, else the NCCL all-to-all).  Reports the per-GPU
    exchange rate against NVLink 5 (900 GB/s per direction) and the wall time."""
    import shutil

    import paper_2604_01949_b200 as R
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    n = 65_536
    path = base / "xchg_in"
    if rank == 0 and not (path / "manifest.json").exists():
        base.mkdir(parents=True, exist_ok=True)
        tmp = base / f".xchg_in.{os.getpid()}"
        R.synth_store(tmp, R.SynthConfig(**dict(CFG5["synth"], n_obs=n)))
        os.replace(tmp, path)
    out = base / f"xchg_out_w{world}"
    if rank == 0:
        shutil.rmtree(out, ignore_errors=True)
    dist.barrier()
    plan = R.plan_shuffle(n, 64, 16_384, 7)
    t0 = time.perf_counter()
    st = R.run_shuffle([path], plan, out, R.ShuffleOutputConfig(4096, 2), device=local, rank=rank, world=world,
                       group=dist.group.WORLD)
    wall = allreduce_max(time.perf_counter() - t0, dist)
    # per GPU: bytes this rank sent to other ranks over the time its exchange took
    send_s = st.send_ms / 1e3 if st.a2a == "ipc" else st.exchange_s
    rate = st.peer_bytes / max(send_s, 1e-12) / 1e9
    rate_min = -allreduce_max(-rate, dist)
    exch_max = allreduce_max(st.exchange_s, dist)
    if rank == 0:
        shutil.rmtree(out, ignore_errors=True)
    payload = sum(f.stat().st_size for f in (path / "shards").iterdir())
    return {"workload": "cfg5-shaped: 65,536 cells x 62,710 genes, ~2k nnz/cell, c=64 m=16,384 (4 rounds), "
                        "out chunk 4096 x 2 per shard (8 shards)",
            "a2a": st.a2a, "value": payload / wall / 1e9, "unit": "GB/s (payload, files -> files, wall, max over ranks)",
            "wall_s": wall, "exchange_s_max": exch_max, "peer_bytes_rank0": st.peer_bytes,
            "roofline": {"bound": "nvlink", "achieved": rate_min, "peak": 900.0, "unit": "GB/s",
                         "frac": rate_min / 900.0, "traffic": None,
                         "peak_source": "NVLink 5 per direction per GPU (nominal)",
                         "kernel": "k_csr_copy_tma record mode storing into peer receive buffers" if st.a2a == "ipc"
                         else "pack into a local send buffer + NCCL all_to_all_single",
                         "achieved_def": "min over ranks of (bytes sent to other ranks / exchange time)"}}


def run_ours_coded(args, wl, rank, world, local, dist):
    """A workload whose verbatim records exceed HBM (cfg2 at 10M cells, 240 GB): the
    store's re-encoded staging image is resident in HBM (resident_coded, ~70 GB) and
    every step runs through the loader -- the fetched blocks expanded device-to-device
    (k_d8_decode) then the batch densified (+ normalize/log1p).  `value` = cells / the
    device time of K such steps (CUDA events on the loader's stream); the roofline is
    the densify kernel's, timed per batch with the loader's kernel events."""
    import torch

    import paper_2604_01949_b200 as R
    torch.cuda.set_device(local)
    W = WORKLOADS[wl]
    reader = R.StoreReader(procedural_spec(W))
    man = reader.manifest()
    K, Wm = args.steps, args.warmup
    t_open = time.perf_counter()
    ds = R.DeviceStore(reader, local, "resident_coded")
    open_s = time.perf_counter() - t_open
    rec_b, img_b = ds.image_bytes()
    stream = torch.cuda.current_stream()
    cfg = R.LoaderConfig(**W["loader"], rank=rank, world=world)
    it = R.BatchIterator(ds, cfg, 0, output="dense", out_dtype=W["out"]["out_dtype"], transform=W["out"]["transform"],
                         out_slots=3, stream=stream, time_kernels=True)
    for _ in range(Wm):
        it.next()
    torch.cuda.synchronize()
    c0 = it.counters()
    clk = Clocks(local).__enter__()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cells = nnz = 0
    for _ in range(K):
        b = it.next()
        cells += b.n_rows
        nnz += b.nnz
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = e0.elapsed_time(e1)
    c1 = it.counters()
    it.close()
    max_ms = allreduce_max(total_ms, dist)
    asm_ms, dec_ms = (c1.assembly_ms - c0.assembly_ms) / K, (c1.decode_ms - c0.decode_ms) / K
    fused = c1.kernels_launched - c0.kernels_launched == K  # K3d: one kernel per step, no decode
    esz = 2 if W["out"]["out_dtype"] == "bf16" else 4
    if fused:
        # densify straight from the staged delta records: read each row's share of its coded
        # record (u8 column deltas, 2-bit top-byte codes, low value bytes; the image's mean
        # bytes per row, which include its indptr / first-column / escape-base entries) and
        # the row ref; write the dense row + gidx
        alg = cells * (img_b / man.n_obs + 16 + man.n_var * esz + 8) / K
        kname = "k_csr_densify_d8 (from the coded staging records, fused normalize+log1p)"
    else:
        # densify over idx16 records (the expanded staging records): read 2 B id + 4 B value
        # per entry, the row ref and the u32 indptr pair; write the dense f32 row + gidx
        alg = (nnz * (2 + 4) + cells * (16 + 8 + man.n_var * esz + 8)) / K
        kname = "k_csr_densify (idx16 records, fused normalize+log1p)"
    peak, peak_src = peaks()
    ds.close()
    e2e = run_e2e(args, wl, reader, W, rank, world, local, dist)
    clk.__exit__(None, None, None)
    if rank != 0:
        return None
    res = {"metric": METRIC, "value": world * cells / (max_ms / 1e3), "unit": "cells/s", "n_gpus": world,
           "steps": K, "warmup": Wm, "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": W["dtype"],
           "data": "synthetic (procedural counts record source == synth_store bytes; never materialised)",
           "config": bench_config(wl, world),
           "details": {"staging": "resident_coded: the store's re-encoded staging image in HBM (%.1f GB for %.1f GB "
                                  "of records); %s" % (img_b / 1e9, rec_b / 1e9, "every step densifies the batch rows straight "
                                  "from their coded records (one kernel)" if fused else "per step the fetched blocks "
                                  "are expanded device-to-device, then the batch is densified"),
                       "open_s": open_s, "decode_ms_per_step": dec_ms, "densify_ms_per_step": asm_ms,
                       "launch": "loader steps (BatchIterator.next), device-timed with CUDA events",
                       "cells_per_step_per_rank": cells / K},
           "roofline": {"bound": "hbm", "achieved": alg / (asm_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": alg / (asm_ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                        "kernel": kname,
                        "alg_bytes_per_launch": alg, "avg_launch_ms": asm_ms},
           "e2e": e2e, "gpu_launches": c1.kernels_launched - c0.kernels_launched, "clocks": clk.summary()}
    if world == 1 and not args.no_cpu_baseline:
        rpath, _ = ensure_ref_store(wl)
        res["cpu_baseline"] = cpu_baseline(rpath, W, threads=1)
    return res


def run_ours(args, wl, rank, world, local, dist):
    import ctypes as C

    import torch

    import paper_2604_01949_b200 as R
    from paper_2604_01949_b200 import _lib as L

    torch.cuda.set_device(local)
    W = WORKLOADS[wl]
    path = ensure_store(wl, rank, world, dist)
    reader = R.StoreReader(path)
    man = reader.manifest()
    K, Wm = args.steps, args.warmup

    # ------------------------------------------------ device-resident value --
    vstaging = W.get("value_staging", "resident")
    ds = R.DeviceStore(reader, local, vstaging)
    onehot = man.layout == "dense" and vstaging == "resident_coded"
    img_gb = ds.image_bytes()[1] / 1e9
    base, offs = ds.arena()
    desc = ds.arena_desc()
    batches = schedule_batches(man.n_obs, W["loader"], rank, world, Wm + K)
    b = W["loader"]["batch_rows"]
    refs = np.zeros((Wm + K, b, 2), np.uint64)
    rows = []
    for i, g in enumerate(batches):
        refs[i, :len(g), 0] = offs[g.astype(np.int64) // man.chunk_rows]
        refs[i, :len(g), 1] = g
        rows.append(len(g))
    # batches per launch (BatchIterator(batches_per_launch=G) does the same): G consecutive
    # batches' rows assembled by one launch into one [G*b, n_var] output; a step is still
    # one batch.  G divides K so that exactly K batches are timed.
    G = max(g for g in range(1, max(1, args.batches_per_launch or W.get("group", 1)) + 1) if K % g == 0)
    launches = [(i, 1) for i in range(Wm)] + [(Wm + j * G, G) for j in range(K // G)]
    d_refs = []
    for s0, g in launches:  # each launch's rows, contiguous
        d_refs.append(torch.from_numpy(np.concatenate([refs[i, :rows[i]] for i in range(s0, s0 + g)]).view(
            np.int64)).cuda())
    esz = {"f32": 4, "bf16": 2, "native": {"f32": 4, "f64": 8, "i32": 4, "u8": 1}[man.value_dtype]}[
        W["out"]["out_dtype"]]
    # a ring of output buffers spanning > 2 x L2 (126 MB): every launch writes its batch
    # rows to HBM, never over the still-cached output of the previous launch
    out_bytes = G * b * man.n_var * esz + 16
    n_out = max(2, -(-(256 << 20) // out_bytes))
    outs = [torch.empty(out_bytes, dtype=torch.uint8, device="cuda") for _ in range(n_out)]
    gouts = [torch.empty(G * b, dtype=torch.int64, device="cuda") for _ in range(n_out)]
    stream = torch.cuda.current_stream()
    od = {"f32": L.F32, "bf16": L.BF16, "native": L.NATIVE}[W["out"]["out_dtype"]]
    xf = L.XF_NORMALIZE_LOG1P if W["out"]["transform"] else L.XF_NONE
    lib = L.lib()

    def launch(j, st=stream):
        n = d_refs[j].shape[0]
        out, gout = outs[j % n_out], gouts[j % n_out]
        if man.layout == "csr":
            rc = lib.rfl_csr_densify(C.byref(desc), d_refs[j].data_ptr(), n, od, xf, 1e4, out.data_ptr(),
                                     gout.data_ptr(), C.c_void_p(st.cuda_stream))
        else:
            fn = lib.rfl_onehot_gather if onehot else lib.rfl_dense_gather
            rc = fn(C.byref(desc), d_refs[j].data_ptr(), n, od, out.data_ptr(), gout.data_ptr(),
                    C.c_void_p(st.cuda_stream))
        L.check(rc)

    KL = K // G  # timed launches
    for i in range(Wm):
        launch(i)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        # the K timed steps captured once as a CUDA graph (one node per batch
        # assembly): back-to-back device execution without host launch gaps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            cap = torch.cuda.current_stream()
            for k in range(KL):
                launch(Wm + k, cap)
        graph.replay()  # upload + warm
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(KL)]
    clk = Clocks(local).__enter__()  # sampled across the value and e2e timed regions (starts with a 250 ms sleep)
    # one more untimed pass right before the timed one, so the GPU is not coming out of
    # the sampler's idle gap (clock / power-state ramp) when the clock starts
    if graph is not None:
        graph.replay()
    else:
        for k in range(KL):
            launch(Wm + k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if graph is not None:
        # a ~100 us device-side spin queued ahead of the start event: the graph launch is
        # submitted while the GPU is busy, so the timed region is the K steps' device time
        # and not also the host's graph-launch latency (~5-10 us, which alone cost cfg4's
        # 2-launch, ~36 us region 0.12 of its roofline fraction)
        torch.cuda._sleep(200_000)
        ev[0][0].record(stream)
        graph.replay()
        ev[-1][1].record(stream)
    else:
        for k in range(KL):
            ev[k][0].record(stream)
            launch(Wm + k)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = ev[0][0].elapsed_time(ev[-1][1])
    per = [total_ms / KL] * KL if graph is not None else [s.elapsed_time(e) for s, e in ev]
    cells = sum(rows[Wm:])
    max_ms = allreduce_max(total_ms, dist)

    # algorithmic bytes per launch: read row refs + indptr pair +
    # indices/values of every nnz; write the dense rows + gidx.
    alg = 0
    if man.layout == "csr":
        isz, vsz = 4 if man.index_dtype == "u32" else 8, {"f32": 4, "f64": 8, "i32": 4, "u8": 1}[man.value_dtype]
        nnz_tot = 0
        rn = _row_nnz(reader, man)
        for i in range(Wm, Wm + K):
            nnz_tot += int(rn[refs[i, :rows[i], 1].astype(np.int64)].sum())
        alg = nnz_tot * (isz + vsz) + cells * (16 + 2 * isz + man.n_var * esz + 8)
    elif onehot:  # read the row's 2-bit codes (n_var / 16 B) + its ref, write the row + gidx
        alg = cells * (16 + man.n_var // 16 + man.n_var * esz + 8)
    else:
        alg = cells * (16 + man.n_var * 1 + man.n_var * esz + 8)
    alg_per_launch = alg / KL
    avg_launch_s = statistics.mean(per) / 1e3
    peak, peak_src = peaks()
    achieved = alg_per_launch / avg_launch_s / 1e9
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_{wl}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")

    # ---------------------------------------------------------------- e2e --
    e2e = run_e2e(args, wl, reader, W, rank, world, local, dist)
    if not args.no_verbatim_e2e and os.environ.get("RIFFLE_E2E_STAGING", "stream_pinned") == "stream_pinned":
        # the same e2e leg with the pinned image left verbatim (no re-encoding at open), for reference
        old_nw = os.environ.get("RFL_NARROW")
        os.environ["RFL_NARROW"] = "0"
        try:
            v = run_e2e(args, wl, reader, W, rank, world, local, dist)
        finally:
            if old_nw is None:
                os.environ.pop("RFL_NARROW", None)
            else:
                os.environ["RFL_NARROW"] = old_nw
        e2e["verbatim_staging"] = {"value": v["value"], "h2d_bytes_per_step": v["h2d_bytes_per_step"],
                                   "open_s": v["open_s"]}
    if not args.no_file_e2e:
        # the out-of-core path: the same e2e leg reading the shard files per fetch (BlockReader
        # read-ahead threads, page cache), nothing pinned up front
        v = run_e2e(args, wl, reader, W, rank, world, local, dist, staging="stream_file")
        e2e["stream_file"] = {"value": v["value"], "h2d_bytes_per_step": v["h2d_bytes_per_step"],
                              "open_s": v["open_s"]}
    clk.__exit__(None, None, None)
    ds.close()

    res = None
    if rank == 0:
        value = world * (cells / K) / (max_ms / K / 1e3)  # whole job: N ranks x cells per step / step time
        res = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": K, "warmup": Wm,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": W["dtype"], "data": "synthetic (product synth_store == reference synth_store bytes)",
            "config": bench_config(wl, world),
            "details": {"staging": ("resident_coded: the store's one-hot staging image in HBM (%.2f GB of 2-bit "
                                    "channel codes for %.2f GB of records), rows written straight from the codes"
                                    % (img_gb, ds_bytes(reader) / 1e9)) if onehot else "resident (chunk records in HBM)",
                        "launch": (f"K/{G} launches ({G} batches each) replayed as one CUDA graph" if graph is not None
                                   else "eager launches"),
                        "l2": "inputs larger than L2 (store %.2f GB); outputs rotate over %d buffers of %.0f MB "
                             "(> 2 x L2), so no launch writes over the cached output of the previous one" % (
                            ds_bytes(reader) / 1e9, n_out, out_bytes / 1e6),
                        "cells_per_step_per_rank": cells / K, "batches_per_launch": G},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "k_csr_densify" if man.layout == "csr" else (
                             "k_onehot_gather" if onehot else "k_dense_gather"),
                         "alg_bytes_per_launch": alg_per_launch, "avg_launch_ms": avg_launch_s * 1e3},
            "e2e": e2e,
            "gpu_launches": KL,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(path, W, threads=1)
    if world > 1 and not args.no_exchange:
        try:
            xr = preshuffle_exchange_leg(rank, world, local, dist)
        except Exception as e:  # reported, not fatal for the loader line
            xr = {"error": f"{type(e).__name__}: {e}"}
        if res is not None:
            res["preshuffle_exchange"] = xr
    return res


def ds_bytes(reader):
    p = Path(reader.root) / "shards"
    return sum(f.stat().st_size for f in p.iterdir())


def _row_nnz(reader, man):
    """Per-row nnz from the records' indptrs (host, for the algorithmic byte count)."""
    out = np.zeros(man.n_obs, np.int64)
    it = np.uint32 if man.index_dtype == "u32" else np.uint64
    for q in range(man.chunk_count()):
        rec = reader.read_record(q)
        rows = int(np.frombuffer(rec, np.uint32, 1, 0)[0])
        ip = np.frombuffer(rec, it, rows + 1, 12).astype(np.int64)
        out[q * man.chunk_rows:q * man.chunk_rows + rows] = np.diff(ip)
    return out


def run_e2e(args, wl, reader, W, rank, world, local, dist, staging=None):
    import torch

    import paper_2604_01949_b200 as R
    K, Wm = args.steps, args.warmup
    # stream_pinned (default) or stream_file (page cache / O_DIRECT reads)
    staging = staging or os.environ.get("RIFFLE_E2E_STAGING", "stream_pinned")
    t_open = time.perf_counter()
    ds = R.DeviceStore(reader, local, staging)  # pin + validate + re-encode (stream_pinned); headers (stream_file)
    open_s = time.perf_counter() - t_open
    rec_b, img_b = ds.image_bytes()
    stream = torch.cuda.current_stream()
    epoch = 0
    # prefetch_depth = read-ahead I/O threads for stream_file (8 of the box's 16 cores: 2.85 M cells/s
    # vs 2.23 M with 16 and 1.32 M with 4, profiles/r2/s3r)
    depth = int(os.environ.get("RIFFLE_E2E_DEPTH", "8" if staging == "stream_file" else "4"))
    cfg = R.LoaderConfig(**W["loader"], prefetch_depth=depth, rank=rank, world=world)

    # batches per launch / per call (BatchIterator(batches_per_launch=G).next_many(G)): a
    # step is still one batch; G steps share one staging copy batch, decode and launch
    G = max(1, args.batches_per_launch or W.get("e2e_group", 1))
    # whole groups only: the warm-up ends on a group boundary and the timed steps are a
    # multiple of G, so every group assembled inside the timed region is counted in full
    Wm = -(-Wm // G) * G
    # workloads with ~10-30 us steps time at least e2e_min_steps of them (a 20-step region
    # would be ~1 ms, dominated by the first group's ramp); the count is in the line
    K = -(-max(K, W.get("e2e_min_steps", 0)) // G) * G

    def make_it(e):
        return R.BatchIterator(ds, cfg, e, output=W["out"]["output"], out_dtype=W["out"]["out_dtype"],
                               transform=W["out"]["transform"], out_slots=3, stream=stream, batches_per_launch=G)

    it = make_it(epoch)
    host = torch.empty(W["loader"]["batch_rows"] * G, dtype=torch.int64).pin_memory()
    host_ptr, stream_h = host.data_ptr(), stream.cuda_stream
    h2d_done = [0]  # bytes staged by iterators already retired
    k_done = [0]    # kernels launched by iterators already retired
    pend = []

    def step():
        nonlocal it, epoch, pend
        if not pend:
            pend = it.next_many(G)
            if not pend:
                h2d_done[0] += it.counters().h2d_bytes
                k_done[0] += it.counters().kernels_launched
                it.close()
                epoch += 1
                it = make_it(epoch)
                pend = it.next_many(G)
            pend.reverse()
        b = pend.pop()
        n = b.n_rows
        b.ids_to_host(host_ptr, stream_h)  # D2H of the step's result ids (one cudaMemcpyAsync)
        return n

    for _ in range(Wm):
        step()
    torch.cuda.synchronize()
    h2d0 = h2d_done[0] + it.counters().h2d_bytes
    k0 = k_done[0] + it.counters().kernels_launched
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record(stream)
    cells = 0
    trace = os.environ.get("RIFFLE_E2E_TRACE")
    for _ in range(K):
        ts = time.perf_counter()
        cells += step()
        if trace:
            print(f"# e2e step host {1e3 * (time.perf_counter() - ts):.3f} ms", file=sys.stderr)
    e_ev.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = s_ev.elapsed_time(e_ev)
    h2d = h2d_done[0] + it.counters().h2d_bytes - h2d0
    launches = k_done[0] + it.counters().kernels_launched - k0
    t_max = allreduce_max(max(ms, wall * 1e3), dist)
    it.close()
    ds.close()
    return {"value": world * cells / (t_max / 1e3), "unit": "cells/s",
            "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": 8 * cells / K, "steps": K, "warmup": Wm,
            "staging": ("stream_pinned (records in pinned host RAM, re-encoded losslessly at open: u8 column "
                        "deltas or u16 ids; each fetched block cudaMemcpyAsync'd, expanded on the GPU)"
                        if staging == "stream_pinned" else
                        "stream_file (BlockReader: prefetch_depth I/O threads pread the fetch order from the shard "
                        "files into pinned buffers; blocks cudaMemcpyAsync'd per fetch)"),
            "api": ("paper_2604_01949_b200.BatchIterator.next -> rfl_loader_next" if G == 1 else
                    f"paper_2604_01949_b200.BatchIterator(batches_per_launch={G}).next_many({G}) -> rfl_loader_next_many"),
            "gpu_launches": launches,
            "open_s": open_s,  # DeviceStore open, outside the timed region: reported, not hidden
            "record_gb": rec_b / 1e9, "staging_image_gb": img_b / 1e9,
            "open_what": ("read, validate and re-encode every record into the page-locked staging image"
                          if staging == "stream_pinned" else "read and check every record header + indptr")}


def cpu_baseline(path, W, threads):
    """The reference's CPU path (oracle/_ref = /root/reference compiled unmodified),
    BatchIterator + to_dense per batch, on a bounded sample (metrics.cpp:99-136 timing)."""
    from oracle.oracle import Ref
    ld = W["loader"]
    dens = W["out"]["output"] == "dense" and W["synth"]["layout"] == "csr"
    nb = int(os.environ.get("RIFFLE_CPU_BATCHES", "0"))
    if nb <= 0:  # size the sample for ~10 s of CPU work from a 4-batch probe (epoch 1, untimed)
        v0, _, _ = Ref.throughput(path, ld["fetch_block_rows"], ld["buffer_capacity_rows"], ld["batch_rows"],
                                  seed=ld["seed"], depth=4, epoch0=1, threads=threads, max_batches=4, densify=dens)
        nb = int(min(200, max(8, 10.0 * v0 / ld["batch_rows"])))
    v, rows, wall = Ref.throughput(path, ld["fetch_block_rows"], ld["buffer_capacity_rows"], ld["batch_rows"],
                                   seed=ld["seed"], depth=4, epoch0=0, threads=threads, max_batches=nb,
                                   densify=dens)
    return {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference",
            "sample": f"{rows} cells = first {nb} batches of epoch(s) 0..{threads - 1} per thread, "
                      f"BatchIterator(prefetch_depth=4){' + to_dense' if dens else ''}, wall {wall:.1f}s",
            "host_cpus": os.cpu_count()}


def run_preshuffle(args, rank, world, local, dist):
    """--workload cfg5: the pre-shuffle (run_shuffle) through the public API.

    A step is one round of the plan (m rows gathered, permuted, packed into
    records and written).  `value`: payload GB/s of the device round pipeline
    (row scan + record pack kernels, CUDA events) -- the records are resident in
    HBM when those kernels run; `e2e`: payload GB/s of the whole run_shuffle
    call (file reads, H2D, kernels, D2H, shard + provenance writes), wall clock,
    max over ranks.  One untimed run_shuffle of the same collection first (warm
    page cache, CUDA context, allocations)."""
    import shutil

    import torch

    import paper_2604_01949_b200 as R
    torch.cuda.set_device(local)
    path = ensure_store("cfg5", rank, world, dist)
    man = R.StoreReader(path).manifest()
    payload = ds_bytes(R.StoreReader(path))
    plan = R.plan_shuffle(man.n_obs, CFG5["c"], CFG5["m"], CFG5["seed"])
    oc = R.ShuffleOutputConfig(CFG5["out_chunk_rows"], CFG5["out_cps"])
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    out = base / f"cfg5_out_w{world}"

    def one():
        if rank == 0:
            shutil.rmtree(out, ignore_errors=True)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        st = R.run_shuffle([path], plan, out, oc, device=local, rank=rank, world=world,
                           group=dist.group.WORLD if dist else None)
        return st, time.perf_counter() - t0

    one()  # warm-up run
    clk = Clocks(local).__enter__()
    st, wall = one()
    clk.__exit__(None, None, None)
    wall_max = allreduce_max(wall, dist)
    # device time of the round pipeline per rank: the pack kernels, plus (N > 1) the
    # exchange phase (peer stores / all-to-all + the barrier that closes it), max over ranks
    gpu_max = allreduce_max(st.gpu_ms + (st.exchange_s * 1e3 if world > 1 else 0.0), dist)
    if rank == 0:
        shutil.rmtree(out, ignore_errors=True)
    if rank != 0:
        return None
    peak, peak_src = peaks()
    nnz = (payload - man.chunk_count() * 12 - 4 * (man.n_obs + man.chunk_count())) / 8  # u32 idx + f32 val
    rounds = st.rounds_executed
    # K5 (+K1) algorithmic bytes over the run: read every entry + row header once, write every
    # encoded entry + indptr once, per rank
    # K5 algorithmic bytes over the run, per rank: read every entry (u32 id + f32 value) and
    # write it once; per row the row ref (16 B) + its prefix entry (8 B) read, the u32
    # indptr entry written.  N=1 runs the pack alone (host-planned prefix); the N>1
    # send side adds the device scan's per-row reads (16 + 2 x 4 B) and prefix write (8 B)
    per_row = 16 + 8 + 4 + (32 if world > 1 else 0)
    alg = (nnz * 16 + man.n_obs * per_row) / world
    res = {"metric": "preshuffle GB/s", "value": payload / (gpu_max / 1e3) / 1e9, "unit": "GB/s",
           "n_gpus": world, "steps": rounds, "warmup": rounds, "ms_per_step": gpu_max / rounds,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32+f32 (bytes)",
           "data": "synthetic (product synth_store == reference synth_store bytes)",
           "config": bench_config("cfg5", world),
           "details": {"payload_GB": payload / 1e9,
                       "value_def": "payload bytes / device time of the round pack kernels (N > 1: + the "
                                    "exchange phase), max over ranks"},
           "roofline": {"bound": "hbm", "achieved": alg / (gpu_max / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": alg / (gpu_max / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                        "kernel": "k_csr_pack (record-mode TMA copy)" + (" + k_row_scan" if world > 1 else ""),
                        "alg_bytes_per_launch": alg / rounds,
                        "avg_launch_ms": gpu_max / rounds},
           "e2e": {"value": payload / wall_max / 1e9, "unit": "GB/s", "h2d_bytes_per_step": st.h2d_bytes / rounds,
                   "d2h_bytes_per_step": st.d2h_bytes / rounds,
                   "api": "paper_2604_01949_b200.run_shuffle -> rfl_run_shuffle", "wall_s": wall_max,
                   "rows_per_s": man.n_obs / wall_max},
           "gpu_launches": (2 if world > 1 else 1) * rounds, "clocks": clk.summary()}
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_shuffle_baseline()
    return res


def cpu_shuffle_baseline():
    """The reference run_shuffle (oracle/_ref, unmodified, single-threaded by design)
    on a bounded subset of the same shape."""
    import shutil

    from oracle.oracle import Ref
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    n = int(os.environ.get("RIFFLE_CFG5_REF_ROWS", CFG5["ref_rows"]))
    sub = base / f"cfg5_ref_{n}"
    if not (sub / "manifest.json").exists():  # the reference's own synth_store (never the product)
        s = CFG5["synth"]
        Ref.synth(sub, n, s["n_var"], s["layout"], s["value_dtype"], s["index_dtype"], s["density"], s["seed"],
                  s["chunk_rows"], s["chunks_per_shard"])
    rout = base / "cfg5_ref_out"
    shutil.rmtree(rout, ignore_errors=True)
    t0 = time.perf_counter()
    Ref.run_shuffle([sub], rout, CFG5["c"], min(CFG5["m"], n), CFG5["seed"], CFG5["out_chunk_rows"], CFG5["out_cps"])
    w = time.perf_counter() - t0
    shutil.rmtree(rout, ignore_errors=True)
    pb = sum(f.stat().st_size for f in (sub / "shards").iterdir())
    return {"value": pb / w / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"run_shuffle of a {n}-row subset of the same shape ({pb / 1e9:.2f} GB), wall {w:.1f}s"}


# --impl reference input sizes: cfg1 is the whole workload (100k cells); the other
# workloads' reference inputs are bounded subsets of the same shape (whole epochs of
# the subset are timed; the per-cell cost does not depend on n_obs)
REF_ROWS = {"cfg1": None, "cfg2": 65_536, "cfg3": 131_072, "cfg4": 524_288}


def ensure_ref_store(wl):
    """The reference arm's input, built without the product: the reference's own
    synth_store (oracle/_ref) for the reference-synth shapes, the oracle's numpy
    restatement of the procedural generators for cfg2 (counts) / cfg4 (one-hot).
    Byte-identical to what the product synthesises for the same config
    (tests/test_host.py, tests/test_oracle.py)."""
    from oracle import oracle as O
    base = Path(os.environ.get("RIFFLE_BENCH_DIR", "/tmp/riffle_bench"))
    s = dict(WORKLOADS[wl]["synth"])
    n = REF_ROWS[wl] or s["n_obs"]
    path = base / f"ref_{wl}_{n}"
    if not (path / "manifest.json").exists():
        base.mkdir(parents=True, exist_ok=True)
        tmp = base / f".ref_{wl}.{os.getpid()}"
        if s.get("counts"):
            O.synth_counts_np(tmp, n, s["n_var"], s["seed"], s["chunk_rows"], s["chunks_per_shard"], s["value_dtype"])
        elif s.get("one_hot"):
            O.synth_one_hot_np(tmp, n, s["n_var"], s["seed"], s["chunk_rows"], s["chunks_per_shard"], s["one_hot"])
        else:
            O.Ref.synth(tmp, n, s["n_var"], s["layout"], s["value_dtype"], s.get("index_dtype", "u32"),
                        s["density"], s["seed"], s["chunk_rows"], s["chunks_per_shard"])
        os.replace(tmp, path)
    return path, n


def bench_config(wl, world):
    """`config` of a bench line: the same keys (and workload) in both arms."""
    if wl == "cfg5":
        return {"workload": CFG5["desc"], "l2": "rounds of ~1 GB of records, larger than L2",
                "parallelism": f"{world} rank(s): rank b mod W stages block b, shard s owned by rank s mod W"}
    W = WORKLOADS[wl]
    return {"workload": W["desc"], "l2": "inputs larger than L2 (the store exceeds 126 MB); the timed launches' "
                                         "outputs rotate over buffers totalling > 2 x L2",
            "parallelism": f"dp{world} (disjoint plan positions per rank, no collective)"}


def run_reference(args, wl, rank, world):
    """--impl reference: the reference CPU implementation (oracle/_ref, the unmodified
    reference compiled from its sources), all host threads, rank 0 only.  Never
    imports the product.  Timed like riffle::run_throughput(epochs=1, warmup=1)
    (metrics.cpp:99-136): every thread drains one whole warm-up epoch, then one
    whole timed epoch (BatchIterator(prefetch_depth=4) + to_dense per CSR batch)."""
    if rank != 0:
        return None
    from oracle.oracle import Ref
    if wl == "cfg5":
        b = cpu_shuffle_baseline()
        return {"metric": "preshuffle GB/s", "value": b["value"], "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32+f32 (bytes)",
                "data": "synthetic (reference synth_store)", "impl": "reference",
                "config": bench_config(wl, world), "threads": 1,
                "cpu_baseline": b, "e2e": {"value": b["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                           "d2h_bytes_per_step": 0}}
    W = WORKLOADS[wl]
    path, n = ensure_ref_store(wl)
    threads = os.cpu_count() or 1
    ld = W["loader"]
    dens = W["out"]["output"] == "dense" and W["synth"]["layout"] == "csr"
    Ref.throughput(path, ld["fetch_block_rows"], ld["buffer_capacity_rows"], ld["batch_rows"], seed=ld["seed"],
                   depth=4, epoch0=1000, threads=threads, max_batches=0, densify=dens)  # warm-up epochs
    v, rows, wall = Ref.throughput(path, ld["fetch_block_rows"], ld["buffer_capacity_rows"], ld["batch_rows"],
                                   seed=ld["seed"], depth=4, epoch0=0, threads=threads, max_batches=0,
                                   densify=dens)
    steps = rows / ld["batch_rows"]
    sample = (f"{threads} concurrent BatchIterators x one whole epoch each (epochs 0..{threads - 1}; one whole "
              f"warm-up epoch each before) over {'the workload store' if REF_ROWS[wl] is None else f'a {n}-row subset of the workload shape'}"
              f" ({rows} cells){' + to_dense' if dens else ''}, wall {wall:.1f}s")
    return {"metric": METRIC, "value": v, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": wall * 1e3 / max(steps, 1e-9), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": W["dtype"],
            "data": "synthetic (reference synth_store; cfg2/cfg4: the oracle's numpy procedural generator)",
            "impl": "reference", "config": bench_config(wl, world), "threads": threads,
            "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg1", choices=sorted(WORKLOADS) + ["cfg5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--no-file-e2e", action="store_true", help="skip the stream_file e2e leg")
    ap.add_argument("--no-exchange", action="store_true", help="N>1: skip the pre-shuffle exchange leg")
    ap.add_argument("--batches-per-launch", type=int, default=0,
                    help="batches assembled per launch (default: the workload's; 1 = one launch per batch)")
    ap.add_argument("--no-verbatim-e2e", action="store_true",
                    help="skip the second e2e leg with the verbatim (not re-encoded) pinned image")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    dist = None
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        local = local % max(ndev, 1)  # more ranks than GPUs only in tests (gloo control plane)
        torch.cuda.set_device(local)
        backend = os.environ.get("RIFFLE_BENCH_BACKEND", "nccl" if ndev >= world else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        res = run_reference(args, args.workload, rank, world)
    elif args.workload == "cfg5":
        res = run_preshuffle(args, rank, world, local, dist)
    elif WORKLOADS[args.workload].get("procedural"):
        res = run_ours_coded(args, args.workload, rank, world, local, dist)
    else:
        res = run_ours(args, args.workload, rank, world, local, dist)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
