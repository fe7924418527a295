"""Generate tests/golden/shapes.json: reference outputs at the BASELINE bench
shapes (the shapes bench.py and profiles/ report), from the compiled reference
(oracle/_ref/libriffle_ref.so, built from /root/reference by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden_shapes.py
Inputs are described by their generator config (the reference synth_store, or
the oracle's numpy procedural generators for the counts / one-hot shapes that
the reference has no generator for); the GPU tests regenerate them with the
product synth, which is byte-identical (tests/test_host.py,
tests/test_oracle.py).  Outputs are pinned by FNV-1a hashes
(tests/test_support.hpp:57-77) of the reference's batches:

* cfg1  100k x 20k CSR, f=64 B=b=4096: the whole of epoch 0 (global_indices,
        CSR MiniBatch, to_dense) -- the full BASELINE config 1 size;
* cfg2  36k-gene counts CSR (2k-4k nnz/cell), f=1024 B=16384 b=4096: MiniBatch
        CSR + to_dense hashes (normalize+log1p is absent from the reference:
        checked against the numpy fp64 restatement on the device side);
* cfg3  dense 12,288-byte u8 rows, f=256 B=16384 b=1024: raw batch hashes and
        hashes of the oracle's exact u8 -> bf16 cast of the reference batches;
* cfg4  dense 4 x 1024 one-hot u8 rows, f=512 B=16384 b=2048: batch hashes;
* cfg5  run_shuffle of a 62,710-gene CSR store with 4,096-row output chunks
        (records > 64 MB): digests of every output file.
"""
from __future__ import annotations

import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import (Orc, Ref, synth_counts_np, synth_one_hot_np,  # noqa: E402
                           u8_to_bf16_bits)

FNV0 = 0xCBF29CE484222325


def fnv(arrs, h=FNV0):
    for a in arrs:
        h = Orc.fnv1a64(np.ascontiguousarray(a), h)
    return h


SHAPES = {
    "cfg1": dict(gen="ref_synth", n_obs=100_000, n_var=20_000, layout="csr", value_dtype="f32", index_dtype="u32",
                 density=0.1, seed=0, chunk_rows=64, cps=128,
                 loader=dict(f=64, B=4096, b=4096, seed=0, epoch=0), want="csr,to_dense"),
    "cfg2": dict(gen="counts", n_obs=12_288, n_var=36_000, layout="csr", value_dtype="f32", index_dtype="u32",
                 seed=1, chunk_rows=1024, cps=8,
                 loader=dict(f=1024, B=16384, b=4096, seed=0, epoch=0), want="csr,to_dense"),
    "cfg3": dict(gen="ref_synth", n_obs=8_192, n_var=12_288, layout="dense", value_dtype="u8", density=0.1,
                 seed=2, chunk_rows=256, cps=16,
                 loader=dict(f=256, B=16384, b=1024, seed=0, epoch=0), want="dense"),
    "cfg4": dict(gen="one_hot", n_obs=20_480, n_var=4096, layout="dense", value_dtype="u8", seed=3,
                 chunk_rows=512, cps=16, one_hot=4,
                 loader=dict(f=512, B=16384, b=2048, seed=0, epoch=0), want="dense"),
}
CFG5 = dict(gen="ref_synth", n_obs=12_288, n_var=62_710, layout="csr", value_dtype="f32", index_dtype="u32",
            density=2000 / 62_710, seed=4, chunk_rows=64, cps=128,
            shuffle=dict(c=64, m=8192, seed=7, out_chunk_rows=4096, out_cps=2))


def make_store(path, s):
    if s["gen"] == "counts":
        synth_counts_np(path, s["n_obs"], s["n_var"], s["seed"], s["chunk_rows"], s["cps"], s["value_dtype"])
    elif s["gen"] == "one_hot":
        synth_one_hot_np(path, s["n_obs"], s["n_var"], s["seed"], s["chunk_rows"], s["cps"], s["one_hot"])
    else:
        Ref.synth(path, s["n_obs"], s["n_var"], s["layout"], s["value_dtype"], s.get("index_dtype", "u32"),
                  s["density"], s["seed"], s["chunk_rows"], s["cps"])


def main():
    g = {"generator": "tests/golden/make_golden_shapes.py over oracle/_ref/libriffle_ref.so (reference proj/core)"}
    tmp = Path(tempfile.mkdtemp(prefix="shapes_"))
    try:
        for name, s in SHAPES.items():
            t0 = time.time()
            make_store(tmp / name, s)
            ld = s["loader"]
            ent = dict(s)
            ent["gidx_fnv"], ent["nnz"], ent["rows"] = [], [], []
            for bt in Ref.iterate(tmp / name, ld["f"], ld["B"], ld["b"], seed=ld["seed"], epoch=ld["epoch"],
                                  want=s["want"]):
                ent["gidx_fnv"].append(hex(fnv([bt["gidx"]])))
                ent["rows"].append(len(bt["gidx"]))
                if s["layout"] == "csr":
                    ent.setdefault("csr_fnv", []).append(hex(fnv([bt["indptr"], bt["indices"], bt["data"]])))
                    ent.setdefault("dense_fnv", []).append(hex(fnv([bt["to_dense"]])))
                    ent["nnz"].append(int(bt["indptr"][-1]))
                else:
                    ent.setdefault("dense_fnv", []).append(hex(fnv([bt["dense"]])))
                    if name == "cfg3":
                        ent.setdefault("bf16_fnv", []).append(hex(fnv([u8_to_bf16_bits(bt["dense"])])))
            ent.update(Ref.last_counters)
            g[name] = ent
            print(f"{name}: {len(ent['rows'])} batches, {time.time() - t0:.1f}s", flush=True)
            shutil.rmtree(tmp / name)
        t0 = time.time()
        make_store(tmp / "cfg5", CFG5)
        sh = CFG5["shuffle"]
        out = tmp / "cfg5_out"
        stats = Ref.run_shuffle([tmp / "cfg5"], out, sh["c"], sh["m"], sh["seed"], sh["out_chunk_rows"],
                                sh["out_cps"])
        files = sorted(p.relative_to(out).as_posix() for p in out.rglob("*") if p.is_file())
        ent = dict(CFG5)
        ent.update(stats)
        ent["files"] = {f: hex(Orc.fnv1a64(np.frombuffer((out / f).read_bytes(), np.uint8))) for f in files}
        ent["sizes"] = {f: (out / f).stat().st_size for f in files}
        g["cfg5"] = ent
        print(f"cfg5: {len(files)} files, {time.time() - t0:.1f}s", flush=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    p = Path(__file__).resolve().parent / "shapes.json"
    p.write_text(json.dumps(g, indent=1) + "\n")
    print(f"wrote {p} ({p.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
