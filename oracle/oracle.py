"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU checker for the B200 hot path.  Two layers:

* ``Ref`` — ctypes over ``oracle/_ref/libriffle_ref.so``: the *unmodified*
  reference C++ library (/root/reference/proj/core) compiled in place by
  ``oracle/Makefile`` behind our flat shim ``oracle/ref_shim.cpp``.
* ``Orc`` + the numpy functions below — our own restatement of the
  reference algorithms (C for the integer schedule in ``riffle_oracle.c``;
  numpy for byte/float arithmetic).  Pinned against ``Ref`` and the golden
  vectors under ``tests/golden/``.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libriffle_ref.so"
ORC_SO = HERE / "_build" / "libriffle_oracle.so"

u64p = C.POINTER(C.c_uint64)

# dtype.hpp:8-16 enum encodings
LAYOUT = {"dense": 0, "csr": 1}
VDT = {"f32": 0, "f64": 1, "i32": 2, "u8": 3}
IDT = {"u32": 0, "u64": 1}
CODEC = {"none": 0, "deflate": 1}
NP_VDT = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "u8": np.uint8}
NP_IDT = {"u32": np.uint32, "u64": np.uint64}


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def build(quiet: bool = True) -> None:
    """Build oracle/_build (our C restatement) and, when /root/reference is
    present, oracle/_ref (the reference).  On the GPU box only prebuilt files
    are used."""
    import subprocess

    targets = ["oracle"]
    if Path("/root/reference/proj/core/src").is_dir():
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", "-C", str(HERE)] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


# ----------------------------------------------------------------------------
# The compiled reference
# ----------------------------------------------------------------------------
class Ref:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
            L = C.CDLL(str(REF_SO))
            L.ref_last_error.restype = C.c_char_p
            L.ref_iter_open.restype = C.c_void_p
            L.ref_iter_open.argtypes = [C.c_char_p] + [C.c_uint64] * 4 + [C.c_uint32, C.c_int, C.c_uint64, C.c_int]
            L.ref_iter_next.argtypes = [C.c_void_p, u64p, u64p]
            for n in ("ref_iter_gidx", "ref_iter_dense", "ref_iter_close"):
                getattr(L, n).argtypes = [C.c_void_p] + ([C.c_void_p] if n != "ref_iter_close" else [])
            L.ref_iter_csr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.ref_iter_to_dense.argtypes = [C.c_void_p, C.c_void_p]
            L.ref_iter_counters.argtypes = [C.c_void_p] + [u64p] * 5
            L.ref_synth.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                    C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
            L.ref_rng_next.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p]
            L.ref_rng_bounded.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
            L.ref_rng_shuffle_iota.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
            L.ref_plan_epoch.argtypes = [C.c_uint64] * 6 + [C.c_void_p, C.c_void_p]
            L.ref_read_rows_csr.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, u64p, u64p,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
            L.ref_read_rows_dense.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
            L.ref_plan_shuffle.argtypes = [C.c_uint64] * 4 + [u64p, C.c_void_p, C.c_void_p]
            L.ref_run_shuffle.argtypes = [C.POINTER(C.c_char_p), C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                          C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                          u64p, u64p]
            L.ref_throughput.restype = C.c_double
            L.ref_throughput.argtypes = [C.c_char_p] + [C.c_uint64] * 4 + [C.c_uint32, C.c_uint64, C.c_uint32,
                                                                          C.c_uint64, C.c_int, u64p,
                                                                          C.POINTER(C.c_double)]
            cls._lib = L
        return cls._lib

    @classmethod
    def err(cls) -> str:
        return cls.lib().ref_last_error().decode()

    @classmethod
    def check(cls, rc: int) -> None:
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {cls.err()}")

    # -- rng
    @classmethod
    def rng_next(cls, seed, n, tag=None):
        out = np.zeros(n, np.uint64)
        cls.lib().ref_rng_next(seed, tag or 0, tag is not None, n, _p(out))
        return out

    @classmethod
    def rng_bounded(cls, seed, bound, n, tag=None):
        out = np.zeros(n, np.uint64)
        cls.lib().ref_rng_bounded(seed, tag or 0, tag is not None, bound, n, _p(out))
        return out

    @classmethod
    def plan_epoch(cls, n_obs, f, B, b, seed, epoch):
        nb = (n_obs + f - 1) // f
        s = np.zeros(nb, np.uint64)
        e = np.zeros(nb, np.uint64)
        cls.check(cls.lib().ref_plan_epoch(n_obs, f, B, b, seed, epoch, _p(s), _p(e)))
        return list(zip(s.tolist(), e.tolist()))

    # -- stores
    @classmethod
    def synth(cls, path, n_obs, n_var, layout="csr", vdtype="f32", idtype="u32", density=0.1,
              seed=0, chunk_rows=64, cps=128, codec="none"):
        cls.check(cls.lib().ref_synth(str(path).encode(), n_obs, n_var, LAYOUT[layout], VDT[vdtype],
                                      IDT[idtype], density, seed, chunk_rows, cps, CODEC[codec]))

    @classmethod
    def read_rows_csr(cls, path, ranges):
        st = np.array([r[0] for r in ranges], np.uint64)
        en = np.array([r[1] for r in ranges], np.uint64)
        rows, nnz = C.c_uint64(), C.c_uint64()
        L = cls.lib()
        cls.check(L.ref_read_rows_csr(str(path).encode(), _p(st), _p(en), len(ranges), C.byref(rows),
                                      C.byref(nnz), None, None, None))
        man = read_manifest(path)
        indptr = np.zeros(rows.value + 1, np.uint64)
        indices = np.zeros(nnz.value, np.uint64)
        data = np.zeros(nnz.value, NP_VDT[man["value_dtype"]])
        cls.check(L.ref_read_rows_csr(str(path).encode(), _p(st), _p(en), len(ranges), C.byref(rows),
                                      C.byref(nnz), _p(indptr), _p(indices), _p(data)))
        return indptr, indices, data

    @classmethod
    def read_rows_dense(cls, path, ranges):
        man = read_manifest(path)
        total = sum(e - s for s, e in ranges)
        st = np.array([r[0] for r in ranges], np.uint64)
        en = np.array([r[1] for r in ranges], np.uint64)
        out = np.zeros((total, man["n_var"]), NP_VDT[man["value_dtype"]])
        cls.check(cls.lib().ref_read_rows_dense(str(path).encode(), _p(st), _p(en), len(ranges), _p(out)))
        return out

    # -- loader
    @classmethod
    def iterate(cls, path, f, B, b, seed=0, epoch=0, depth=0, drop_last=False, want="gidx", cache_bypass=False):
        """Yields per batch: dict(gidx=..., [indptr, indices, data] | [dense] | [to_dense]).

        want: "gidx" | "csr" | "dense" | "to_dense" (comma separated allowed)."""
        L = cls.lib()
        man = read_manifest(path)
        h = L.ref_iter_open(str(path).encode(), f, B, b, seed, depth, int(drop_last), epoch, int(cache_bypass))
        if not h:
            raise RuntimeError(cls.err())
        wants = set(want.split(","))
        vdt = NP_VDT[man["value_dtype"]]
        try:
            while True:
                n, nnz = C.c_uint64(), C.c_uint64()
                rc = L.ref_iter_next(h, C.byref(n), C.byref(nnz))
                if rc == 0:
                    break
                if rc < 0:
                    raise RuntimeError(cls.err())
                out = {}
                g = np.zeros(n.value, np.uint64)
                L.ref_iter_gidx(h, _p(g))
                out["gidx"] = g
                if "csr" in wants:
                    ip = np.zeros(n.value + 1, np.uint64)
                    ix = np.zeros(nnz.value, np.uint64)
                    dv = np.zeros(nnz.value, vdt)
                    L.ref_iter_csr(h, _p(ip), _p(ix), _p(dv))
                    out.update(indptr=ip, indices=ix, data=dv)
                if "dense" in wants:
                    dv = np.zeros((n.value, man["n_var"]), vdt)
                    L.ref_iter_dense(h, _p(dv))
                    out["dense"] = dv
                if "to_dense" in wants:
                    dv = np.zeros((n.value, man["n_var"]), vdt)
                    cls.check(L.ref_iter_to_dense(h, _p(dv)))
                    out["to_dense"] = dv
                yield out
            cnt = [C.c_uint64() for _ in range(5)]
            L.ref_iter_counters(h, *[C.byref(c) for c in cnt])
            cls.last_counters = dict(zip(["blocks_fetched", "peak_buffer_rows", "read_ops", "bytes_read",
                                          "chunks_decoded"], [c.value for c in cnt]))
        finally:
            L.ref_iter_close(h)

    # -- preshuffle
    @classmethod
    def plan_shuffle(cls, total, c, m, seed):
        nr = C.c_uint64()
        L = cls.lib()
        cls.check(L.ref_plan_shuffle(total, c, m, seed, C.byref(nr), None, None))
        nb = (total + c - 1) // c
        lens = np.zeros(max(nr.value, 1), np.uint64)
        ids = np.zeros(max(nb, 1), np.uint64)
        cls.check(L.ref_plan_shuffle(total, c, m, seed, C.byref(nr), _p(lens), _p(ids)))
        out, k = [], 0
        for r in range(nr.value):
            out.append(ids[k:k + int(lens[r])].tolist())
            k += int(lens[r])
        return out

    @classmethod
    def run_shuffle(cls, in_paths, out_path, c, m, seed, out_chunk_rows, out_cps, outer=True, out_idt=None,
                    codec="none"):
        arr = (C.c_char_p * len(in_paths))(*[str(p).encode() for p in in_paths])
        peak, rounds = C.c_uint64(), C.c_uint64()
        cls.check(cls.lib().ref_run_shuffle(arr, len(in_paths), int(outer), c, m, seed, str(out_path).encode(),
                                            out_chunk_rows, out_cps, -1 if out_idt is None else IDT[out_idt],
                                            CODEC[codec], C.byref(peak), C.byref(rounds)))
        return {"peak_resident_rows": peak.value, "rounds": rounds.value}

    @classmethod
    def throughput(cls, path, f, B, b, seed=0, depth=4, epoch0=0, threads=1, max_batches=0, densify=True):
        rows, wall = C.c_uint64(), C.c_double()
        v = cls.lib().ref_throughput(str(path).encode(), f, B, b, seed, depth, epoch0, threads, max_batches,
                                     int(densify), C.byref(rows), C.byref(wall))
        if v < 0:
            raise RuntimeError(cls.err())
        return v, rows.value, wall.value


# ----------------------------------------------------------------------------
# Our C restatement (riffle_oracle.c)
# ----------------------------------------------------------------------------
class Orc:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ORC_SO.exists():
                build()
            L = C.CDLL(str(ORC_SO))
            L.orc_mix64.restype = C.c_uint64
            L.orc_mix64.argtypes = [C.c_uint64]
            L.orc_rng_next.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p]
            L.orc_rng_bounded.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
            L.orc_plan_epoch_ids.argtypes = [C.c_uint64] * 4 + [C.c_void_p]
            L.orc_replay_epoch.restype = C.c_int64
            L.orc_replay_epoch.argtypes = [C.c_uint64] * 6 + [C.c_int, C.c_uint64, C.c_uint64] + [C.c_void_p] * 2 + [u64p] * 3
            L.orc_plan_shuffle.restype = C.c_int64
            L.orc_plan_shuffle.argtypes = [C.c_uint64] * 4 + [C.c_void_p, C.c_void_p]
            L.orc_shuffle_order.argtypes = [C.c_uint64] * 4 + [C.c_void_p]
            L.orc_fnv1a64.restype = C.c_uint64
            L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
            cls._lib = L
        return cls._lib

    @classmethod
    def rng_next(cls, seed, n, tag=None):
        out = np.zeros(n, np.uint64)
        cls.lib().orc_rng_next(seed, tag or 0, tag is not None, n, _p(out))
        return out

    @classmethod
    def rng_bounded(cls, seed, bound, n, tag=None):
        out = np.zeros(n, np.uint64)
        cls.lib().orc_rng_bounded(seed, tag or 0, tag is not None, bound, n, _p(out))
        return out

    @classmethod
    def plan_epoch(cls, n_obs, f, seed, epoch):
        nb = (n_obs + f - 1) // f
        ids = np.zeros(nb, np.uint64)
        cls.lib().orc_plan_epoch_ids(n_obs, f, seed, epoch, _p(ids))
        return [(int(i) * f, min(n_obs, (int(i) + 1) * f)) for i in ids]

    @classmethod
    def replay_epoch(cls, n_obs, f, B, b, seed=0, epoch=0, drop_last=False, rank=0, world=1):
        """Returns (list of per-batch gidx arrays, peak, blocks)."""
        g = np.zeros(max(n_obs, 1), np.uint64)
        lens = np.zeros((n_obs + b - 1) // b + 2, np.uint64)
        rows, peak, blocks = C.c_uint64(), C.c_uint64(), C.c_uint64()
        nb = cls.lib().orc_replay_epoch(n_obs, f, B, b, seed, epoch, int(drop_last), rank, world, _p(g), _p(lens),
                                        C.byref(rows), C.byref(peak), C.byref(blocks))
        if nb < 0:
            raise ValueError("invalid loader config")
        out, k = [], 0
        for i in range(nb):
            out.append(g[k:k + int(lens[i])].copy())
            k += int(lens[i])
        return out, peak.value, blocks.value

    @classmethod
    def plan_shuffle(cls, total, c, m, seed):
        nb = (total + c - 1) // c
        lens = np.zeros(max(nb, 1), np.uint64)
        ids = np.zeros(max(nb, 1), np.uint64)
        nr = cls.lib().orc_plan_shuffle(total, c, m, seed, _p(lens), _p(ids))
        if nr < 0:
            raise ValueError("invalid shuffle plan")
        out, k = [], 0
        for r in range(nr):
            out.append(ids[k:k + int(lens[r])].tolist())
            k += int(lens[r])
        return out

    @classmethod
    def shuffle_order(cls, total, c, m, seed):
        out = np.zeros(max(total, 1), np.uint64)
        if cls.lib().orc_shuffle_order(total, c, m, seed, _p(out)) != 0:
            raise ValueError("invalid shuffle plan")
        return out[:total]

    @classmethod
    def fnv1a64(cls, arr: np.ndarray, h: int = 0xcbf29ce484222325) -> int:
        a = np.ascontiguousarray(arr)
        return cls.lib().orc_fnv1a64(_p(a), a.nbytes, h)


# ----------------------------------------------------------------------------
# numpy restatement of the store format and the byte/float kernels
# ----------------------------------------------------------------------------
def read_manifest(path) -> dict:
    """manifest.cpp:49-97 (JSON keys in field order)."""
    return json.loads((Path(path) / "manifest.json").read_text())


def _shard_footer(p: Path, slots: int):
    """shard.hpp:13-19, shard.cpp:18-54: records, then (u64 off, u64 len) x slots, then SHRDIDX1."""
    raw = p.read_bytes()
    tail = slots * 16 + 8
    assert raw[-8:] == b"SHRDIDX1", f"bad magic in {p}"
    foot = np.frombuffer(raw[len(raw) - tail:len(raw) - 8], np.uint64).reshape(slots, 2)
    return raw, foot


def read_chunk_records(path) -> list[bytes]:
    """All chunk records of a store in chunk order (codec none)."""
    man = read_manifest(path)
    n_chunks = (man["n_obs"] + man["chunk_rows"] - 1) // man["chunk_rows"]
    cps = man["chunks_per_shard"]
    out = []
    for s in range((n_chunks + cps - 1) // cps):
        raw, foot = _shard_footer(Path(path) / "shards" / f"s{s:08d}.bin", cps)
        for k in range(cps):
            if s * cps + k >= n_chunks:
                break
            off, ln = int(foot[k, 0]), int(foot[k, 1])
            out.append(raw[off:off + ln])
    return out


def decode_csr_record(rec: bytes, idt: str, vdt: str):
    """store.cpp:52-64,81-122: [n_rows u32][nnz u64][indptr (rows+1)][indices nnz][data nnz]."""
    rows, nnz = struct.unpack_from("<IQ", rec, 0)
    it, vt = np.dtype(NP_IDT[idt]), np.dtype(NP_VDT[vdt])
    pos = 12
    indptr = np.frombuffer(rec, it, rows + 1, pos).astype(np.uint64)
    pos += (rows + 1) * it.itemsize
    indices = np.frombuffer(rec, it, nnz, pos).astype(np.uint64)
    pos += nnz * it.itemsize
    data = np.frombuffer(rec, vt, nnz, pos)
    return indptr, indices, data


def load_csr_store(path):
    """Whole store as one CSR (indptr u64, indices u64, data)."""
    man = read_manifest(path)
    ips, ixs, dvs, base = [np.zeros(1, np.uint64)], [], [], 0
    for rec in read_chunk_records(path):
        ip, ix, dv = decode_csr_record(rec, man["index_dtype"], man["value_dtype"])
        ips.append(ip[1:] + np.uint64(base))
        ixs.append(ix)
        dvs.append(dv)
        base += int(ip[-1])
    return np.concatenate(ips), np.concatenate(ixs) if ixs else np.zeros(0, np.uint64), np.concatenate(dvs)


def load_dense_store(path) -> np.ndarray:
    man = read_manifest(path)
    recs = read_chunk_records(path)
    return np.frombuffer(b"".join(recs), NP_VDT[man["value_dtype"]]).reshape(man["n_obs"], man["n_var"])


def csr_gather(indptr, indices, data, rows):
    """CsrBuffer::take → batch append (loader.cpp:145-154): rows in order, rebased indptr."""
    rows = np.asarray(rows, np.int64)
    lo, hi = indptr[rows].astype(np.int64), indptr[rows + 1].astype(np.int64)
    nnz = hi - lo
    out_ip = np.zeros(len(rows) + 1, np.uint64)
    out_ip[1:] = np.cumsum(nnz)
    sel = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)]) if len(rows) else np.zeros(0, np.int64)
    return out_ip, indices[sel], data[sel]


def to_dense(indptr, indices, data, n_var) -> np.ndarray:
    """block.cpp:135-146: zero matrix, then each nnz copied to [r, idx]."""
    n = len(indptr) - 1
    out = np.zeros((n, n_var), data.dtype)
    r = np.repeat(np.arange(n), np.diff(indptr.astype(np.int64)))
    out[r, indices.astype(np.int64)] = data
    return out


def normalize_log1p(dense: np.ndarray, target: float = 1e4) -> np.ndarray:
    """New (absent from the reference): y = log1p(x * T / Σ_row x),
    Σ in fp64; a row with Σ = 0 stays 0.  Returned in fp64 (the checker)."""
    x = dense.astype(np.float64)
    s = x.sum(axis=1, keepdims=True)
    scale = np.where(s != 0, target / np.where(s != 0, s, 1.0), 0.0)
    return np.log1p(x * scale)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 → bf16 (bit pattern as uint16); NaN stays quiet NaN."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    nan = np.isnan(x)
    out = rounded.astype(np.uint16)
    out[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return out


def u8_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """u8 → bf16 is exact (≤ 255 needs 8 significant bits)."""
    return f32_to_bf16_bits(x.astype(np.float32))


def write_csr_store(path, indptr, indices, data, n_var, chunk_rows, cps, idt="u32", vdt="f32"):
    """StoreWriter restatement for hand-built CSR stores (store.cpp:140-297, shard.cpp:76-103):
    lets tests build stores the synth cannot (empty rows, huge rows, u64 ids)."""
    p = Path(path)
    (p / "shards").mkdir(parents=True)
    n = len(indptr) - 1
    it, vt = np.dtype(NP_IDT[idt]), np.dtype(NP_VDT[vdt])
    recs = []
    for s in range(0, n, chunk_rows):
        e = min(n, s + chunk_rows)
        lo, hi = int(indptr[s]), int(indptr[e])
        ip = (np.asarray(indptr[s:e + 1], np.uint64) - np.uint64(lo)).astype(it)
        rec = struct.pack("<IQ", e - s, hi - lo) + ip.tobytes() + np.asarray(indices[lo:hi]).astype(it).tobytes() \
            + np.asarray(data[lo:hi]).astype(vt).tobytes()
        recs.append(rec)
    for sh in range((len(recs) + cps - 1) // cps):
        part = recs[sh * cps:(sh + 1) * cps]
        body, slots, off = b"", [], 0
        for r in part:
            slots.append((off, len(r)))
            body += r
            off += len(r)
        slots += [(2**64 - 1, 2**64 - 1)] * (cps - len(part))
        foot = b"".join(struct.pack("<QQ", a, b) for a, b in slots) + b"SHRDIDX1"
        (p / "shards" / f"s{sh:08d}.bin").write_bytes(body + foot)
    names = ",\n".join(f'    "v{i}"' for i in range(n_var))
    man = ('{\n  "format_version": 1,\n  "layout": "csr",\n  "n_obs": %d,\n  "n_var": %d,\n  "value_dtype": "%s",\n'
           '  "index_dtype": "%s",\n  "chunk_rows": %d,\n  "chunks_per_shard": %d,\n  "codec": "none",\n'
           '  "var_names": %s,\n  "has_provenance": false\n}\n') % (
        n, n_var, vdt, idt, chunk_rows, cps, ("[\n" + names + "\n  ]") if n_var else "[]")
    (p / "manifest.json").write_text(man)


# ----------------------------------------------------------------------------
# Procedural synthetic stores (numpy restatement of the product's synth_counts /
# synth_one_hot): the reference has no such generator, so bench.py's
# --impl reference leg builds its cfg2 / cfg4 inputs with these (never with the
# product).  Pinned byte-for-byte against the product synth in tests/test_host.py.
# ----------------------------------------------------------------------------
_M1, _M2, _GOLD = np.uint64(0xbf58476d1ce4e5b9), np.uint64(0x94d049bb133111eb), np.uint64(0x9e3779b97f4a7c15)


def mix64_np(x) -> np.ndarray:
    """rng.hpp:12-17 (splitmix64 finalizer), elementwise over uint64 (wrapping)."""
    x = np.asarray(x, np.uint64) + _GOLD
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def synth_counts_np(path, n_obs, n_var, seed, chunk_rows, cps, vdt="f32"):
    """Counts-like CSR (2,000 + h mod 2,001 stratified columns per row, values 1..64)."""
    sd = np.uint64(seed)
    rows = np.arange(n_obs, dtype=np.uint64)
    h = mix64_np(sd ^ mix64_np(rows))
    nnz = np.minimum(np.uint64(n_var), np.uint64(2000) + h % np.uint64(2001)).astype(np.int64)
    indptr = np.zeros(n_obs + 1, np.uint64)
    indptr[1:] = np.cumsum(nnz)
    r = np.repeat(np.arange(n_obs), nnz)
    k = (np.arange(int(indptr[-1]), dtype=np.int64) - indptr[r].astype(np.int64)).astype(np.uint64)
    n = nnz[r].astype(np.uint64)
    hr = h[r]
    lo = k * np.uint64(n_var) // n
    hi = (k + np.uint64(1)) * np.uint64(n_var) // n
    idx = lo + mix64_np(hr ^ k) % (hi - lo)
    cnt = np.uint64(1) + mix64_np(hr ^ (k + np.uint64(1 << 32))) % np.uint64(64)
    data = cnt.astype(np.float32) if vdt == "f32" else cnt.astype(np.int32)
    write_csr_store(path, indptr, idx, data, n_var, chunk_rows, cps, "u32", vdt)


def write_dense_store(path, x: np.ndarray, chunk_rows, cps, vdt="u8"):
    """StoreWriter restatement for dense stores (row-major records, store.cpp:31-33)."""
    p = Path(path)
    (p / "shards").mkdir(parents=True)
    n, n_var = x.shape
    recs = [np.ascontiguousarray(x[s:s + chunk_rows]).tobytes() for s in range(0, n, chunk_rows)]
    for sh in range((len(recs) + cps - 1) // cps):
        part = recs[sh * cps:(sh + 1) * cps]
        slots, off = [], 0
        with open(p / "shards" / f"s{sh:08d}.bin", "wb") as f:
            for r in part:
                slots.append((off, len(r)))
                f.write(r)
                off += len(r)
            slots += [(2**64 - 1, 2**64 - 1)] * (cps - len(part))
            f.write(b"".join(struct.pack("<QQ", a, b) for a, b in slots) + b"SHRDIDX1")
    names = ",\n".join(f'    "v{i}"' for i in range(n_var))
    man = ('{\n  "format_version": 1,\n  "layout": "dense",\n  "n_obs": %d,\n  "n_var": %d,\n  "value_dtype": "%s",\n'
           '  "chunk_rows": %d,\n  "chunks_per_shard": %d,\n  "codec": "none",\n'
           '  "var_names": %s,\n  "has_provenance": false\n}\n') % (
        n, n_var, vdt, chunk_rows, cps, ("[\n" + names + "\n  ]") if n_var else "[]")
    (p / "manifest.json").write_text(man)


def synth_one_hot_np(path, n_obs, n_var, seed, chunk_rows, cps, channels=4):
    """One-hot dense u8 rows: position p of row i is 1 in channel mix64(h_i ^ p) % channels."""
    L = n_var // channels
    x = np.zeros((n_obs, n_var), np.uint8)
    p = np.arange(L, dtype=np.uint64)
    for s in range(0, n_obs, 65536):
        e = min(n_obs, s + 65536)
        h = mix64_np(np.uint64(seed) ^ mix64_np(np.arange(s, e, dtype=np.uint64)))
        ch = (mix64_np(h[:, None] ^ p[None, :]) % np.uint64(channels)).astype(np.int64)
        rr = np.arange(e - s)[:, None]
        x[s + rr, ch * L + p[None, :].astype(np.int64)] = 1
    write_dense_store(path, x, chunk_rows, cps, "u8")
