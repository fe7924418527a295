"""Generate tests/golden/golden.json from the compiled reference
(oracle/_ref/libriffle_ref.so, built from /root/reference by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The committed JSON is what travels to the GPU box.  Stores are described by
their synth_store config (the product synth is byte-identical to the
reference, checked by tests/test_host.py), so fixtures stay small: batch
contents are pinned by FNV-1a hashes (tests/test_support.hpp:57-77).
"""
from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Orc, Ref, read_manifest  # noqa: E402

FNV0 = 0xCBF29CE484222325


def fnv(arrs, h=FNV0):
    for a in arrs:
        h = Orc.fnv1a64(np.ascontiguousarray(a), h)
    return h


STORES = {
    "csr_small": dict(n_obs=3000, n_var=400, layout="csr", value_dtype="f32", index_dtype="u32", density=0.05,
                      seed=11, chunk_rows=64, cps=8),
    "csr_unaligned": dict(n_obs=2501, n_var=257, layout="csr", value_dtype="f32", index_dtype="u32", density=0.1,
                          seed=5, chunk_rows=100, cps=3),
    "csr_u64_f64": dict(n_obs=1200, n_var=130, layout="csr", value_dtype="f64", index_dtype="u64", density=0.2,
                        seed=7, chunk_rows=50, cps=4),
    "dense_u8": dict(n_obs=2000, n_var=192, layout="dense", value_dtype="u8", density=0.1, seed=2, chunk_rows=64,
                     cps=4),
    "dense_f32": dict(n_obs=777, n_var=33, layout="dense", value_dtype="f32", density=0.1, seed=4, chunk_rows=40,
                      cps=5),
}

LOADERS = [  # (store, f, B, b, seed, epoch, drop_last)
    ("csr_small", 64, 512, 256, 0, 0, False),
    ("csr_small", 64, 512, 256, 0, 1, False),
    ("csr_small", 32, 100, 64, 3, 0, True),
    ("csr_unaligned", 70, 300, 128, 9, 2, False),
    ("csr_unaligned", 1, 2501, 500, 1, 0, False),
    ("csr_u64_f64", 25, 200, 100, 4, 0, False),
    ("dense_u8", 256, 1024, 128, 0, 0, False),
    ("dense_f32", 7, 50, 33, 2, 3, False),
]


def synth(path, c):
    Ref.synth(path, c["n_obs"], c["n_var"], c["layout"], c["value_dtype"], c.get("index_dtype", "u32"),
              c["density"], c["seed"], c["chunk_rows"], c["cps"])


def main():
    g = {"generator": "tests/golden/make_golden.py over oracle/_ref/libriffle_ref.so (reference proj/core)"}
    g["rng_next_seed0"] = [hex(x) for x in Ref.rng_next(0, 8)]
    g["rng_bounded_seed42_stream1_4096"] = Ref.rng_bounded(42, 4096, 16, tag=1).tolist()
    g["rng_bounded_seed7_stream3_5"] = Ref.rng_bounded(7, 5, 16, tag=3).tolist()
    g["plan_epoch"] = [
        {"n_obs": n, "f": f, "seed": s, "epoch": e, "blocks": Ref.plan_epoch(n, f, f, 1, s, e)}
        for (n, f, s, e) in [(10, 4, 0, 0), (10, 16, 0, 0), (1000, 64, 5, 3), (97, 10, 1, 1)]
    ]
    g["plan_shuffle"] = [
        {"total": t, "c": c, "m": m, "seed": s, "rounds": Ref.plan_shuffle(t, c, m, s)}
        for (t, c, m, s) in [(100, 10, 30, 0), (10, 10, 10, 0), (1003, 17, 200, 9), (64, 1, 64, 2)]
    ]
    g["stores"] = STORES
    tmp = Path(tempfile.mkdtemp())
    for name, c in STORES.items():
        synth(tmp / name, c)
    loaders = []
    for (st, f, B, b, seed, ep, dl) in LOADERS:
        man = read_manifest(tmp / st)
        want = "csr,to_dense" if man["layout"] == "csr" else "dense"
        batches = list(Ref.iterate(tmp / st, f, B, b, seed=seed, epoch=ep, drop_last=dl, want=want))
        ent = {"store": st, "f": f, "B": B, "b": b, "seed": seed, "epoch": ep, "drop_last": dl,
               "gidx": [bt["gidx"].tolist() for bt in batches], **Ref.last_counters}
        if man["layout"] == "csr":
            ent["csr_fnv"] = [hex(fnv([bt["indptr"], bt["indices"], bt["data"]])) for bt in batches]
            ent["dense_fnv"] = [hex(fnv([bt["to_dense"]])) for bt in batches]
            ent["nnz"] = [int(bt["indptr"][-1]) for bt in batches]
        else:
            ent["dense_fnv"] = [hex(fnv([bt["dense"]])) for bt in batches]
        loaders.append(ent)
    g["loaders"] = loaders
    # reference read_rows (uneven-slice concatenation), store.cpp:590-614
    rr = []
    for st, ranges in [("csr_unaligned", [(150, 420), (7, 8), (2400, 2501), (1000, 1100)]),
                       ("csr_small", [(0, 3000)]), ("csr_u64_f64", [(49, 51), (1199, 1200), (100, 350)])]:
        ip, ix, dv = Ref.read_rows_csr(tmp / st, ranges)
        rr.append({"store": st, "ranges": ranges, "nnz": int(ip[-1]), "fnv": hex(fnv([ip, ix, dv]))})
    g["read_rows_csr"] = rr
    # reference run_shuffle: provenance order == index-computable shuffle order
    sh = []
    for st, c, m, seed, ocr, ocps in [("csr_small", 64, 512, 7, 100, 4), ("csr_unaligned", 17, 300, 3, 64, 2),
                                      ("dense_u8", 32, 256, 1, 128, 3)]:
        out = tmp / f"shuf_{st}"
        stats = Ref.run_shuffle([tmp / st], out, c, m, seed, ocr, ocps)
        files = sorted(p.relative_to(out).as_posix() for p in out.rglob("*") if p.is_file())
        digests = {f: hex(Orc.fnv1a64(np.frombuffer((out / f).read_bytes(), np.uint8))) for f in files}
        sh.append({"store": st, "c": c, "m": m, "seed": seed, "out_chunk_rows": ocr, "out_cps": ocps,
                   **stats, "files": digests})
    g["run_shuffle"] = sh
    out = Path(__file__).resolve().parent / "golden.json"
    out.write_text(json.dumps(g, indent=1) + "\n")
    print(f"wrote {out} ({out.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
