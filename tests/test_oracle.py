"""The CPU oracle, pinned: our C restatement (oracle/riffle_oracle.c) against the
compiled reference (oracle/_ref) and the golden vectors it produced."""
import numpy as np
import pytest

from oracle.oracle import Orc, Ref, load_csr_store, load_dense_store, read_manifest, csr_gather, to_dense

from conftest import fnv


def test_rng_golden(golden):
    assert [hex(x) for x in Orc.rng_next(0, 8)] == golden["rng_next_seed0"]
    # SURVEY §8a a1 golden values
    assert Orc.rng_next(0, 4).tolist() == [0x422EA740D0977210, 0xE062B061B42E2928, 0x5A071FC5930841B6,
                                           0x01334EF8ED3CC2BD]
    assert Orc.rng_bounded(42, 4096, 6, tag=1).tolist() == [1203, 699, 1684, 3085, 260, 1516]
    assert Orc.rng_bounded(42, 4096, 16, tag=1).tolist() == golden["rng_bounded_seed42_stream1_4096"]
    assert Orc.rng_bounded(7, 5, 16, tag=3).tolist() == golden["rng_bounded_seed7_stream3_5"]


@pytest.mark.parametrize("seed,tag,bound", [(0, 0, 1), (1, 2, 3), (99, 7, 2**63 + 5), (5, 11, 1000)])
def test_rng_vs_reference(seed, tag, bound):
    assert (Orc.rng_next(seed, 64, tag=tag) == Ref.rng_next(seed, 64, tag=tag)).all()
    assert (Orc.rng_bounded(seed, bound, 64, tag=tag) == Ref.rng_bounded(seed, bound, 64, tag=tag)).all()


def test_plan_epoch_golden(golden):
    assert Orc.plan_epoch(10, 4, 0, 0) == [(8, 10), (0, 4), (4, 8)]
    for p in golden["plan_epoch"]:
        assert [list(x) for x in Orc.plan_epoch(p["n_obs"], p["f"], p["seed"], p["epoch"])] == p["blocks"]


def test_plan_shuffle_golden(golden):
    assert Orc.plan_shuffle(100, 10, 30, 0) == [[2, 5, 0], [9, 1, 3], [8, 4, 6], [7]]
    for p in golden["plan_shuffle"]:
        assert Orc.plan_shuffle(p["total"], p["c"], p["m"], p["seed"]) == p["rounds"]


def test_replay_golden(golden):
    for ld in golden["loaders"]:
        st = golden["stores"][ld["store"]]
        batches, peak, blocks = Orc.replay_epoch(st["n_obs"], ld["f"], ld["B"], ld["b"], ld["seed"], ld["epoch"],
                                                 ld["drop_last"])
        assert [b.tolist() for b in batches] == ld["gidx"]
        assert blocks == ld["blocks_fetched"]
        assert peak == ld["peak_buffer_rows"]


SWEEP = [(n, f, B, b, s, e, dl) for (n, f, B, b) in [(1, 1, 1, 1), (10, 4, 8, 4), (100, 7, 20, 20), (1000, 64, 64, 1),
                                                       (1000, 1, 1000, 999), (777, 50, 333, 100), (64, 64, 4096, 64)]
         for s in (0, 5) for e in (0, 2) for dl in (False, True)]


@pytest.mark.parametrize("n,f,B,b,seed,epoch,dl", SWEEP)
def test_replay_vs_reference_iterator(tmp_path_factory, n, f, B, b, seed, epoch, dl):
    """Index-only replay == reference BatchIterator global_indices (dense store, any f/B/b)."""
    d = tmp_path_factory.getbasetemp() / f"dense_{n}"
    if not (d / "manifest.json").exists():
        Ref.synth(d, n, 2, "dense", "f32", density=0.1, seed=1, chunk_rows=13, cps=3)
    ref = [bt["gidx"].tolist() for bt in Ref.iterate(d, f, B, b, seed=seed, epoch=epoch, drop_last=dl)]
    got, peak, blocks = Orc.replay_epoch(n, f, B, b, seed, epoch, dl)
    assert [g.tolist() for g in got] == ref
    assert peak == Ref.last_counters["peak_buffer_rows"]
    assert blocks == Ref.last_counters["blocks_fetched"]


def test_numpy_restatement_vs_reference(golden, golden_stores):
    """Our numpy store reader + gather + to_dense reproduce reference batches bit-for-bit."""
    for ld in golden["loaders"]:
        path = golden_stores[ld["store"]]
        man = read_manifest(path)
        if man["layout"] == "csr":
            ip, ix, dv = load_csr_store(path)
            for g, hc, hd in zip(ld["gidx"], ld["csr_fnv"], ld["dense_fnv"]):
                bi, bx, bd = csr_gather(ip, ix, dv, g)
                assert hex(fnv([bi, bx, bd])) == hc
                assert hex(fnv([to_dense(bi, bx, bd, man["n_var"])])) == hd
        else:
            X = load_dense_store(path)
            for g, hd in zip(ld["gidx"], ld["dense_fnv"]):
                assert hex(fnv([np.ascontiguousarray(X[np.asarray(g, np.int64)])])) == hd


def test_shuffle_order_matches_reference_provenance(tmp_path):
    """run_shuffle output order is index-computable: provenance == Orc.shuffle_order."""
    Ref.synth(tmp_path / "in", 1000, 3, "dense", "f32", seed=4, chunk_rows=32, cps=2)
    Ref.run_shuffle([tmp_path / "in"], tmp_path / "out", 17, 200, 9, 64, 3)
    # provenance sidecar shares the store's chunk grid: read its shard records directly
    man = read_manifest(tmp_path / "out")
    import struct
    from pathlib import Path
    rows = []
    n_chunks = (man["n_obs"] + man["chunk_rows"] - 1) // man["chunk_rows"]
    cps = man["chunks_per_shard"]
    for s in range((n_chunks + cps - 1) // cps):
        raw = (Path(tmp_path) / "out" / "provenance" / "shards" / f"s{s:08d}.bin").read_bytes()
        foot = np.frombuffer(raw[len(raw) - cps * 16 - 8:len(raw) - 8], np.uint64).reshape(cps, 2)
        for k in range(cps):
            if s * cps + k >= n_chunks:
                break
            off, ln = int(foot[k, 0]), int(foot[k, 1])
            for i in range(ln // 12):
                ds, src = struct.unpack_from("<IQ", raw, off + 12 * i)
                rows.append(src)
    assert rows == Orc.shuffle_order(1000, 17, 200, 9).tolist()


def test_normalize_and_bf16_restatements():
    from oracle.oracle import normalize_log1p, f32_to_bf16_bits
    x = np.array([[0, 1, 3], [0, 0, 0], [2, 2, 0]], np.float32)
    y = normalize_log1p(x, 1e4)
    assert y[1].tolist() == [0, 0, 0]
    assert np.allclose(y[0], np.log1p(np.array([0, 2500, 7500.0])))
    # RNE: 1 + 2^-8 ties to even (1.0), 1 + 3*2^-8 rounds up
    bits = f32_to_bf16_bits(np.array([1.0, 1 + 2**-8, 1 + 3 * 2**-8, -2.5], np.float32))
    assert bits.tolist() == [0x3F80, 0x3F80, 0x3F82, 0xC020]
