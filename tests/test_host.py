"""CPU tests of the product's host side, all through the C-ABI (no GPU calls):
the library loads and exports every symbol include/riffle_b200.h declares, the
host schedule replays the reference bit-exactly, synth_store is byte-identical,
and store validation raises the reference's error types."""
import filecmp
import os
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2604_01949_b200 as R
from paper_2604_01949_b200 import _lib as L
from oracle.oracle import Orc, Ref

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "riffle_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:rfl_status|const char\*|int|void)\s+(rfl_\w+)\s*\(", header, re.M))
    assert len(declared) >= 25
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == {s[0] for s in L.SIGNATURES}
    assert lib.rfl_version().startswith(b"riffle_b200")


def test_ids_download_argument_checks():
    """rfl_ids_download_async: null buffers with rows to copy are EINVAL (checked
    before any CUDA call); zero rows is a no-op."""
    lib = L.lib()
    assert lib.rfl_ids_download_async(None, 4, None, None) == L.EINVAL
    assert b"null" in lib.rfl_last_error()
    assert lib.rfl_ids_download_async(None, 0, None, None) == L.OK


def test_no_gpu_here_fails_loudly(tmp_path):
    """No CPU fallback: on a GPU-less host, device entry points raise CudaError."""
    if L.lib().rfl_device_count() > 0:
        pytest.skip("GPU present")
    R.synth_store(tmp_path / "s", R.SynthConfig(100, 10, "csr", density=0.2, chunk_rows=10))
    with pytest.raises(R.CudaError):
        R.DeviceStore(tmp_path / "s")


@pytest.mark.parametrize("case", [
    dict(n_obs=10000, n_var=500, layout="csr", value_dtype="f32", index_dtype="u32", density=0.05, seed=3,
         chunk_rows=100, cps=7),
    dict(n_obs=9000, n_var=37, layout="dense", value_dtype="u8", density=0.1, seed=1, chunk_rows=64, cps=4),
    dict(n_obs=5000, n_var=300, layout="csr", value_dtype="f64", index_dtype="u64", density=0.2, seed=9,
         chunk_rows=333, cps=2),
    dict(n_obs=4100, n_var=50, layout="csr", value_dtype="i32", index_dtype="u32", density=1.0, seed=2,
         chunk_rows=4096, cps=1),
    dict(n_obs=1, n_var=1, layout="csr", value_dtype="u8", index_dtype="u32", density=1.0, seed=0, chunk_rows=1,
         cps=1),
    dict(n_obs=300, n_var=5, layout="dense", value_dtype="i32", density=0.1, seed=8, chunk_rows=7, cps=3),
    # Codec::deflate stores (codec.cpp:16-36, one raw DEFLATE stream per record)
    dict(n_obs=3000, n_var=300, layout="csr", value_dtype="f32", index_dtype="u32", density=0.1, seed=5,
         chunk_rows=64, cps=8, codec="deflate"),
    dict(n_obs=2000, n_var=96, layout="dense", value_dtype="u8", density=0.1, seed=6, chunk_rows=50, cps=3,
         codec="deflate"),
    dict(n_obs=1500, n_var=200, layout="csr", value_dtype="f64", index_dtype="u64", density=0.2, seed=4,
         chunk_rows=128, cps=4, codec="deflate"),
])
def test_synth_byte_identical(tmp_path, case):
    c = case
    Ref.synth(tmp_path / "ref", c["n_obs"], c["n_var"], c["layout"], c["value_dtype"], c.get("index_dtype", "u32"),
              c["density"], c["seed"], c["chunk_rows"], c["cps"], codec=c.get("codec", "none"))
    R.synth_store(tmp_path / "gpu", R.SynthConfig(c["n_obs"], c["n_var"], c["layout"], c["value_dtype"],
                                                  c.get("index_dtype", "u32"), c["density"], c["seed"],
                                                  c["chunk_rows"], c["cps"], codec=c.get("codec", "none"),
                                                  threads=3))
    a = sorted(os.listdir(tmp_path / "ref" / "shards"))
    assert a == sorted(os.listdir(tmp_path / "gpu" / "shards"))
    for f in a:
        assert filecmp.cmp(tmp_path / "ref" / "shards" / f, tmp_path / "gpu" / "shards" / f, shallow=False), f
    assert (tmp_path / "ref" / "manifest.json").read_bytes() == (tmp_path / "gpu" / "manifest.json").read_bytes()


def test_store_reader_and_records(golden_stores, golden):
    r = R.StoreReader(golden_stores["csr_small"])
    m = r.manifest()
    c = golden["stores"]["csr_small"]
    assert (m.n_obs, m.n_var, m.layout, m.value_dtype, m.index_dtype, m.chunk_rows) == \
        (c["n_obs"], c["n_var"], "csr", "f32", "u32", c["chunk_rows"])
    from oracle.oracle import read_chunk_records
    recs = read_chunk_records(golden_stores["csr_small"])
    assert len(recs) == m.chunk_count()
    for q in (0, 5, m.chunk_count() - 1):
        assert r.read_record(q) == recs[q]


def test_store_errors(tmp_path):
    with pytest.raises(R.IoError):
        R.StoreReader(tmp_path / "absent")
    R.synth_store(tmp_path / "s", R.SynthConfig(200, 10, "csr", density=0.3, chunk_rows=16, chunks_per_shard=4))
    r = R.StoreReader(tmp_path / "s")
    # truncated shard -> CorruptStore naming the shard (test_store.cpp:405-415)
    p = tmp_path / "s" / "shards" / "s00000001.bin"
    p.write_bytes(p.read_bytes()[:40])
    with pytest.raises(R.CorruptStore, match="truncated|magic"):
        r.read_record(5)
    # a store that exists already is not clobbered (store.cpp:220-222)
    with pytest.raises(R.InvalidArgument):
        R.synth_store(tmp_path / "s", R.SynthConfig(10, 10, "csr", density=0.3))
    # invalid manifest
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "manifest.json").write_text("{\"format_version\": 2}")
    with pytest.raises(R.InvalidArgument):
        R.StoreReader(tmp_path / "bad")
    (tmp_path / "bad" / "manifest.json").write_text("{not json")
    with pytest.raises(R.CorruptStore):
        R.StoreReader(tmp_path / "bad")


def test_loader_config_validate():
    R.LoaderConfig(4, 8, 8).validate()
    for bad in [R.LoaderConfig(0, 8, 1), R.LoaderConfig(8, 4, 1), R.LoaderConfig(4, 8, 9), R.LoaderConfig(4, 8, 0),
                R.LoaderConfig(4, 8, 4, rank=2, world=2)]:
        with pytest.raises(R.InvalidArgument):
            bad.validate()
    with pytest.raises(R.InvalidArgument):
        R.plan_epoch(0, R.LoaderConfig(4, 8, 4), 0)


def test_plan_epoch_matches(golden):
    for p in golden["plan_epoch"]:
        cfg = R.LoaderConfig(p["f"], p["f"], 1, p["seed"])
        assert [list(b) for b in R.plan_epoch(p["n_obs"], cfg, p["epoch"]).blocks] == p["blocks"]


def test_schedule_golden(golden):
    for ld in golden["loaders"]:
        n = golden["stores"][ld["store"]]["n_obs"]
        s = R.EpochSchedule(n, R.LoaderConfig(ld["f"], ld["B"], ld["b"], ld["seed"], drop_last=ld["drop_last"]),
                            ld["epoch"])
        assert [g.tolist() for g in s] == ld["gidx"]
        assert s.next() is None  # idempotent end of epoch
        st = s.stats()
        assert st["peak_buffer_rows"] == ld["peak_buffer_rows"] and st["blocks_fetched"] == ld["blocks_fetched"]


@pytest.mark.parametrize("n,f,B,b,seed,epoch,dl,world", [
    (1, 1, 1, 1, 0, 0, False, 1), (10, 4, 8, 4, 0, 0, False, 1), (1000, 3, 50, 50, 7, 1, True, 1),
    (100000, 64, 4096, 4096, 0, 0, False, 1), (99999, 1024, 16384, 4096, 1, 3, False, 1),
    (5000, 64, 512, 128, 2, 0, False, 2), (5000, 64, 512, 128, 2, 0, True, 4), (7777, 100, 100, 100, 9, 5, False, 8),
])
def test_schedule_vs_oracle(n, f, B, b, seed, epoch, dl, world):
    cfgs = [R.LoaderConfig(f, B, b, seed, drop_last=dl, rank=k, world=world) for k in range(world)]
    allg = []
    for k, cfg in enumerate(cfgs):
        got = [g.tolist() for g in R.EpochSchedule(n, cfg, epoch)]
        exp, _, _ = Orc.replay_epoch(n, f, B, b, seed, epoch, dl, k, world)
        assert got == [e.tolist() for e in exp]
        allg += sum(got, [])
    if not dl:  # epoch completeness across ranks (SPEC acceptance 4)
        assert sorted(allg) == list(range(n))


@pytest.mark.parametrize("n,f,B,b,dl,world", [(5000, 64, 512, 128, False, 3), (7777, 100, 100, 100, False, 8),
                                                (30011, 64, 1024, 500, True, 4), (4096, 64, 512, 512, False, 2)])
def test_even_batches_truncates_to_the_shortest_rank(n, f, B, b, dl, world):
    """even_batches (new, DDP-safe epochs): every rank yields the minimum per-rank
    batch count, and its batches are exactly the first ones of its plain schedule."""
    plain = [list(R.EpochSchedule(n, R.LoaderConfig(f, B, b, 5, drop_last=dl, rank=k, world=world), 1))
             for k in range(world)]
    even = [list(R.EpochSchedule(n, R.LoaderConfig(f, B, b, 5, drop_last=dl, rank=k, world=world,
                                                   even_batches=True), 1)) for k in range(world)]
    m = min(len(p) for p in plain)
    assert all(len(e) == m for e in even)
    for p, e in zip(plain, even):
        assert all((x == y).all() for x, y in zip(p, e))
    one = list(R.EpochSchedule(n, R.LoaderConfig(f, B, b, 5, drop_last=dl, even_batches=True), 1))
    ref = list(R.EpochSchedule(n, R.LoaderConfig(f, B, b, 5, drop_last=dl), 1))
    assert len(one) == len(ref)  # world == 1: the reference schedule


def test_allocation_failure_maps_to_out_of_memory():
    """std::bad_alloc crosses the C-ABI as RFL_ENOMEM -> OutOfMemory (a MemoryError)."""
    with pytest.raises(MemoryError):
        R.EpochSchedule(1 << 44, R.LoaderConfig(1, 1, 1), 0)


def test_schedule_reference_large():
    """The 24-config survey probe at cfg1 scale: replay == reference iterator."""
    import tempfile
    d = Path(tempfile.mkdtemp())
    Ref.synth(d / "s", 20000, 2, "dense", "u8", seed=1, chunk_rows=64, cps=128)
    ref = [bt["gidx"] for bt in Ref.iterate(d / "s", 64, 4096, 4096, seed=42)]
    got = list(R.EpochSchedule(20000, R.LoaderConfig(64, 4096, 4096, 42), 0))
    assert len(got) == len(ref) == 5
    assert all((a == b).all() for a, b in zip(got, ref))


def test_plan_shuffle_and_order(golden):
    for p in golden["plan_shuffle"]:
        assert R.plan_shuffle(p["total"], p["c"], p["m"], p["seed"]).rounds == p["rounds"]
    for (t, c, m, s) in [(1000, 17, 200, 9), (5, 5, 5, 0), (4097, 64, 1024, 3)]:
        assert (R.shuffle_order(t, c, m, s) == Orc.shuffle_order(t, c, m, s)).all()
    with pytest.raises(R.InvalidArgument):
        R.plan_shuffle(10, 0, 5, 0)
    with pytest.raises(R.InvalidArgument):
        R.plan_shuffle(10, 6, 5, 0)


def test_synth_one_hot_store(tmp_path):
    """SynthConfig.one_hot (BASELINE config 4's WGS windows, not in the reference):
    an ordinary dense u8 store (the reference reads it), every row one-hot over
    the channel planes, deterministic in the seed."""
    import paper_2604_01949_b200 as R
    from oracle.oracle import Ref, load_dense_store
    cfgs = dict(n_obs=200, n_var=4 * 32, layout="dense", value_dtype="u8", seed=5, chunk_rows=48,
                chunks_per_shard=2, one_hot=4)
    R.synth_store(tmp_path / "a", R.SynthConfig(**cfgs))
    R.synth_store(tmp_path / "b", R.SynthConfig(**cfgs))
    x = load_dense_store(tmp_path / "a").reshape(200, 4, 32)
    assert ((x == 0) | (x == 1)).all() and (x.sum(axis=1) == 1).all()
    assert (load_dense_store(tmp_path / "b") == load_dense_store(tmp_path / "a")).all()
    # the reference loader reads it like any dense store
    ref = list(Ref.iterate(tmp_path / "a", 48, 96, 50, seed=1, want="dense"))
    for b in ref:
        assert b["dense"].tobytes() == x.reshape(200, 128)[b["gidx"].astype(np.int64)].tobytes()
    with pytest.raises(R.InvalidArgument):
        R.synth_store(tmp_path / "c", R.SynthConfig(**dict(cfgs, n_var=30)))


@pytest.mark.parametrize("kind", ["counts", "one_hot"])
def test_procedural_synth_matches_oracle_generator(tmp_path, kind):
    """The product's procedural generators (cfg2 counts, cfg4 one-hot)
    are byte-identical to the oracle's numpy restatement, which bench.py's
    --impl reference leg and tests/golden/make_golden_shapes.py use."""
    import paper_2604_01949_b200 as R
    from oracle.oracle import synth_counts_np, synth_one_hot_np
    if kind == "counts":
        R.synth_store(tmp_path / "a", R.SynthConfig(1100, 36_000, "csr", "f32", seed=1, chunk_rows=256,
                                                    chunks_per_shard=3, counts=True))
        synth_counts_np(tmp_path / "b", 1100, 36_000, 1, 256, 3)
    else:
        R.synth_store(tmp_path / "a", R.SynthConfig(900, 4096, "dense", "u8", seed=3, chunk_rows=128,
                                                    chunks_per_shard=4, one_hot=4))
        synth_one_hot_np(tmp_path / "b", 900, 4096, 3, 128, 4)
    fa = sorted(p.relative_to(tmp_path / "a") for p in (tmp_path / "a").rglob("*") if p.is_file())
    fb = sorted(p.relative_to(tmp_path / "b") for p in (tmp_path / "b").rglob("*") if p.is_file())
    assert fa == fb
    for f in fa:
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f


def test_procedural_store_matches_synth_files(tmp_path):
    """A "procedural:counts?..." store (records generated on demand, never
    materialised -- bench.py's 240 GB config 2) reads exactly like the files
    synth_store writes for the same config: manifest, record slots, raw records."""
    import paper_2604_01949_b200 as R
    R.synth_store(tmp_path / "a", R.SynthConfig(5000, 36_000, "csr", "f32", seed=1, chunk_rows=1024,
                                                chunks_per_shard=2, counts=True))
    a = R.StoreReader(tmp_path / "a")
    p = R.StoreReader("procedural:counts?n_obs=5000&n_var=36000&seed=1&chunk_rows=1024&chunks_per_shard=2")
    assert a.manifest() == p.manifest()
    assert all(a.read_record(q) == p.read_record(q) for q in range(a.manifest().chunk_count()))
    with pytest.raises(R.InvalidArgument):
        R.StoreReader("procedural:counts?n_obs=10&n_var=x")
    with pytest.raises(R.InvalidArgument):
        R.StoreReader("procedural:gaussian?n_obs=10&n_var=10")
