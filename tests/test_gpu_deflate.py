"""Codec::deflate stores on the GPU path (reference codec.cpp:16-107,
store.cpp:81-122): records are inflated on the host -- at open for the
resident / pinned images, in the read-ahead threads for stream_file -- and the
device assembles batches from the decoded records.  Everything is compared with
the live reference (oracle/_ref) on the same deflate stores: batches, counters
(bytes_read counts the stored, encoded bytes), the CorruptStore text of a
damaged stream, and byte-identical run_shuffle outputs with codec deflate."""
import os
from pathlib import Path

import numpy as np
import pytest

import paper_2604_01949_b200 as R
from oracle.oracle import Ref

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

STORES = {
    "csr_f32": dict(n_obs=3000, n_var=300, layout="csr", vdt="f32", idt="u32", density=0.1, seed=5, cr=64, cps=8),
    "csr_f64_u64": dict(n_obs=1500, n_var=200, layout="csr", vdt="f64", idt="u64", density=0.2, seed=4, cr=128,
                        cps=4),
    "dense_u8": dict(n_obs=2000, n_var=96, layout="dense", vdt="u8", idt="u32", density=0.1, seed=6, cr=50, cps=3),
}


@pytest.fixture(scope="module")
def stores(tmp_path_factory):
    d = tmp_path_factory.mktemp("deflate")
    out = {}
    for k, s in STORES.items():
        Ref.synth(d / k, s["n_obs"], s["n_var"], s["layout"], s["vdt"], s["idt"], s["density"], s["seed"], s["cr"],
                  s["cps"], codec="deflate")
        out[k] = d / k
    return out


@pytest.mark.parametrize("staging,depth,bypass", [("resident", 0, False), ("stream_pinned", 2, False),
                                                  ("stream_file", 0, False), ("stream_file", 3, True)])
@pytest.mark.parametrize("name", list(STORES))
def test_deflate_batches_vs_reference(stores, name, staging, depth, bypass):
    s = STORES[name]
    path = stores[name]
    f, B, b = 70, 400, 128
    want = "csr,to_dense" if s["layout"] == "csr" else "dense"
    ref = list(Ref.iterate(path, f, B, b, seed=3, epoch=1, want=want, cache_bypass=bypass))
    rc = dict(Ref.last_counters)
    outs = ["csr", "dense"] if s["layout"] == "csr" else ["dense"]
    for out in outs:
        it = R.BatchIterator(path, R.LoaderConfig(f, B, b, 3, prefetch_depth=depth, cache_bypass=bypass), 1,
                             staging=staging, output=out)
        got = [x.to_minibatch() for x in it]
        assert len(got) == len(ref)
        for r, m in zip(ref, got):
            assert (m.global_indices == r["gidx"]).all()
            if out == "csr":
                assert (m.block.indptr == r["indptr"]).all() and (m.block.indices == r["indices"]).all()
                assert m.block.data.tobytes() == r["data"].tobytes()
            else:
                assert m.block.values.tobytes() == (r["to_dense"] if s["layout"] == "csr" else r["dense"]).tobytes()
        c = it.counters()
        assert c.blocks_fetched == rc["blocks_fetched"] and c.peak_buffer_rows == rc["peak_buffer_rows"]
        assert (c.read_ops, c.bytes_read, c.chunks_decoded) == (rc["read_ops"], rc["bytes_read"],
                                                                rc["chunks_decoded"])
        it.close()


def _damage(path):
    """Flip bytes inside the first record's DEFLATE stream (test_store.cpp:417-437)."""
    shard = sorted((Path(path) / "shards").iterdir())[0]
    raw = bytearray(shard.read_bytes())
    raw[6:10] = bytes([0x13, 0x37, 0x13, 0x37])
    shard.write_bytes(bytes(raw))


@pytest.mark.parametrize("layout", ["csr", "dense"])
@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
def test_corrupt_deflate_names_the_chunk(tmp_path, layout, staging):
    Ref.synth(tmp_path / "s", 200, 40, layout, "f32", "u32", 0.3, 1, 16, 4, codec="deflate")
    _damage(tmp_path / "s")
    with pytest.raises(RuntimeError) as ref:
        Ref.read_rows_csr(tmp_path / "s", [(0, 200)]) if layout == "csr" else \
            Ref.read_rows_dense(tmp_path / "s", [(0, 200)])
    assert "chunk" in str(ref.value)
    if staging == "stream_file" and layout == "dense":
        # dense records: lengths come from the manifest, so the damage surfaces at fetch
        it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(16, 64, 32, 0, prefetch_depth=2), 0,
                             staging="stream_file")
        with pytest.raises(R.IoError) as ours:
            for _ in it:
                pass
        msg = str(ours.value)
        assert "fetch block [" in msg and msg.split("): ", 1)[1] in str(ref.value)
        return
    with pytest.raises(R.CorruptStore) as ours:
        R.DeviceStore(tmp_path / "s", 0, staging)
    assert "chunk 0" in str(ours.value) and str(ours.value) in str(ref.value)


@pytest.mark.parametrize("in_codec,out_codec", [("deflate", "deflate"), ("deflate", "none"), ("none", "deflate")])
def test_shuffle_deflate_byte_identical(tmp_path, in_codec, out_codec):
    """run_shuffle with deflate members and/or ShuffleOutputConfig.codec = deflate:
    output store + provenance sidecar byte-identical to the reference's."""
    a, b = tmp_path / "a", tmp_path / "b"
    Ref.synth(a, 700, 90, "csr", "f32", "u32", 0.1, 1, 32, 4, codec=in_codec)
    Ref.synth(b, 333, 90, "csr", "f32", "u32", 0.2, 2, 50, 2, codec=in_codec)
    Ref.run_shuffle([a, b], tmp_path / "ref", 16, 200, 5, 77, 3, codec=out_codec)
    plan = R.plan_shuffle(1033, 16, 200, 5)
    R.run_shuffle([a, b], plan, tmp_path / "gpu", R.ShuffleOutputConfig(77, 3, codec=out_codec))
    fa = sorted(p.relative_to(tmp_path / "ref").as_posix() for p in (tmp_path / "ref").rglob("*") if p.is_file())
    fb = sorted(p.relative_to(tmp_path / "gpu").as_posix() for p in (tmp_path / "gpu").rglob("*") if p.is_file())
    assert fa == fb
    for f in fa:
        assert (tmp_path / "ref" / f).read_bytes() == (tmp_path / "gpu" / f).read_bytes(), f


def test_shuffle_deflate_dense(tmp_path):
    Ref.synth(tmp_path / "in", 900, 33, "dense", "u8", "u32", 0.1, 3, 40, 5, codec="deflate")
    Ref.run_shuffle([tmp_path / "in"], tmp_path / "ref", 20, 150, 2, 64, 3, codec="deflate")
    R.run_shuffle([tmp_path / "in"], R.plan_shuffle(900, 20, 150, 2), tmp_path / "gpu",
                  R.ShuffleOutputConfig(64, 3, codec="deflate"))
    for p in sorted((tmp_path / "ref").rglob("*")):
        if p.is_file():
            assert p.read_bytes() == (tmp_path / "gpu" / p.relative_to(tmp_path / "ref")).read_bytes(), p
