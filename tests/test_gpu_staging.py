"""The re-encoded pinned staging image ("Narrowed staging image"):
delta records (u8 column deltas), idx16 records and the verbatim image must all
give the reference's batches bit for bit.  The store is built so that every
boundary is hit: n_var = 65,536 (largest column id 65,535 still fits u16), a
gap of exactly 255 (delta) next to records with a gap of 256 (idx16 fallback),
empty rows, single-entry rows, first columns at 0 and at 65,535."""
import os

import numpy as np
import pytest
import torch

import paper_2604_01949_b200 as R
from oracle.oracle import csr_gather, load_csr_store, normalize_log1p, to_dense, write_csr_store

pytestmark = pytest.mark.gpu

NV = 65536


def _rows(rng, n):
    rows = []
    for i in range(n):
        kind = i % 7
        if kind == 0:
            cols = []                                        # empty row
        elif kind == 1:
            cols = [NV - 1]                                  # single entry at the last column
        elif kind == 2:
            cols = [0, 255, 510, 765]                        # gaps of exactly 255
        elif kind == 3 and (i // 7) % 3 == 0:
            cols = [5, 261, 300, 65535]                      # a gap of 256 (and 65,235): idx16 record
        else:
            start = int(rng.integers(0, NV - 12000))
            gaps = rng.integers(1, 256, int(rng.integers(20, 40)))
            cols = list(start + np.cumsum(gaps))
        rows.append(np.asarray(cols, np.uint64))
    return rows


def _build(tmp_path_factory, vdt):
    rng = np.random.default_rng(7)
    rows = _rows(rng, 336)
    ip = np.zeros(len(rows) + 1, np.uint64)
    ip[1:] = np.cumsum([len(r) for r in rows])
    ix = np.concatenate(rows).astype(np.uint64)
    if vdt == "u8":
        dv = rng.integers(1, 256, len(ix)).astype(np.uint8)
    elif vdt == "f32wide":  # mostly (0.25, 1.25), 12 % anywhere from -1e8 to 1e8: top-byte escapes
        dv = (rng.random(len(ix)) + 0.25).astype(np.float32)
        wide = rng.random(len(ix)) < 0.12
        dv[wide] = (rng.standard_normal(wide.sum()) * 10.0 ** rng.integers(-8, 9, wide.sum())).astype(np.float32)
        dv[::97] = 0.0
        vdt = "f32"
    else:
        dv = (rng.random(len(ix)) + 0.25).astype(np.float32 if vdt == "f32" else np.float64)
    path = tmp_path_factory.mktemp("staging_" + str(dv.dtype)) / "s"
    write_csr_store(path, ip, ix, dv, NV, 16, 8, vdt=vdt)
    return path, ip, ix, dv


@pytest.fixture(scope="module")
def crafted(tmp_path_factory):
    return _build(tmp_path_factory, "f32")


@pytest.mark.parametrize("vdt", ["u8", "f64", "f32wide"])
def test_staging_value_widths(tmp_path_factory, vdt):
    """1- and 8-byte values through the delta staging (value region copied
    word-wise with a byte tail / 8-B aligned in the expanded record), and f32
    values whose top bytes need the escape list of the coded value layout."""
    path, ip, ix, dv = _build(tmp_path_factory, vdt)
    ds = R.DeviceStore(path, 0, "stream_pinned")
    for out in ("csr", "dense"):
        it = R.BatchIterator(ds, R.LoaderConfig(16, 96, 40, 5), 0, output=out)
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if out == "csr":
                mb = b.to_minibatch()
                assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
                assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
            else:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, NV).tobytes()
        assert it.counters().h2d_bytes < it.counters().bytes_read
        it.close()
    ds.close()


@pytest.mark.parametrize("mode", ["delta", "16", "0"])
def test_staging_encodings_bit_exact(crafted, mode):
    path, ip, ix, dv = crafted
    old = os.environ.get("RFL_NARROW")
    if mode != "delta":
        os.environ["RFL_NARROW"] = mode
    try:
        ds = R.DeviceStore(path, 0, "stream_pinned")
    finally:
        if old is None:
            os.environ.pop("RFL_NARROW", None)
        else:
            os.environ["RFL_NARROW"] = old
    cfg = R.LoaderConfig(16, 96, 40, 3)
    for out, xf in (("csr", None), ("dense", None), ("dense", "normalize_log1p")):
        it = R.BatchIterator(ds, cfg, 1, output=out, transform=xf)
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if out == "csr":
                mb = b.to_minibatch()
                assert (np.asarray(mb.block.indptr, np.uint64) == eip).all()
                assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
                assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
            elif xf is None:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, NV).tobytes()
            else:
                want = normalize_log1p(to_dense(eip, eix, edv, NV))
                np.testing.assert_allclose(b.data.cpu().numpy().astype(np.float64), want, rtol=1e-6, atol=0)
        c = it.counters()
        if mode == "0":
            assert c.h2d_bytes >= c.bytes_read  # verbatim records (+ row refs)
        else:
            assert c.h2d_bytes < c.bytes_read
        it.close()
    ds.close()
    torch.cuda.synchronize()


@pytest.mark.parametrize("staging", ["stream_pinned", "resident_coded"])
@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("out_dtype", ["native", "bf16"])
def test_one_hot_dense_staging(tmp_path, out_dtype, fused, staging, monkeypatch):
    """BASELINE config 4's one-hot windows: a dense u8 store whose rows are one-hot
    over 4 channel planes stages as 2-bit codes (16x fewer PCIe bytes) and is
    rebuilt on the GPU -- by K4o straight from the codes (default) or by
    k_d8_decode + the dense gather (RFL_FUSED=0); batches equal the reference's
    row gather bit for bit, 3 batches per launch included.  A single non-one-hot
    byte anywhere keeps the verbatim image (resident_coded then refuses)."""
    monkeypatch.setenv("RFL_FUSED", fused)
    from oracle.oracle import load_dense_store, u8_to_bf16_bits
    for broken in (False, True):
        path = tmp_path / f"oh{int(broken)}"
        R.synth_store(path, R.SynthConfig(n_obs=700, n_var=4 * 64, layout="dense", value_dtype="u8", seed=11,
                                          chunk_rows=32, chunks_per_shard=8, one_hot=4))
        if broken:  # flip one byte of one record in place
            shard = sorted((path / "shards").iterdir())[1]
            raw = bytearray(shard.read_bytes())
            raw[100] = 2
            shard.write_bytes(bytes(raw))
        x = load_dense_store(path).reshape(700, 256)
        if broken and staging == "resident_coded":
            with pytest.raises(R.InvalidArgument):
                R.DeviceStore(path, 0, staging)
            continue
        ds = R.DeviceStore(path, 0, staging)
        it = R.BatchIterator(ds, R.LoaderConfig(32, 160, 64, 9), 0, output="dense", out_dtype=out_dtype,
                             batches_per_launch=3)
        n = 0
        for b in it:
            g = b.global_indices_host.astype(np.int64)
            want = x[g]
            if out_dtype == "bf16":
                got = b.data.view(torch.int16).cpu().numpy().view(np.uint16)
                assert (got == u8_to_bf16_bits(want)).all()
            else:
                assert b.data.cpu().numpy().tobytes() == want.tobytes()
            n += len(g)
        assert n == 700
        c = it.counters()
        if broken:
            assert c.h2d_bytes >= c.bytes_read
        elif staging == "stream_pinned":
            assert c.h2d_bytes < c.bytes_read / 4  # codes are 1/16 of the rows; row refs (16 B) on top
        if not broken:  # 11 batches in 4 groups of <= 3: K4o is one launch per group, no decode
            if fused == "1" and staging == "resident_coded":
                assert c.kernels_launched == 4
            elif fused == "1":  # + one staging pull kernel per group that fetched blocks
                assert 4 < c.kernels_launched <= 8
            else:
                assert c.kernels_launched > 4  # + the decode launches
        it.close()
        ds.close()


def test_wide_axis_keeps_verbatim_staging(tmp_path):
    """n_var > 65,536: column ids do not fit u16, the pinned image stays verbatim
    (and u64 index stores likewise) -- batches still bit-exact."""
    rng = np.random.default_rng(3)
    nv = 70_000
    rows = [np.sort(rng.choice(nv, int(rng.integers(0, 30)), replace=False)).astype(np.uint64) for _ in range(120)]
    ip = np.zeros(len(rows) + 1, np.uint64)
    ip[1:] = np.cumsum([len(r) for r in rows])
    ix = np.concatenate(rows)
    dv = (rng.random(len(ix)) + 0.5).astype(np.float32)
    for idt in ("u32", "u64"):
        path = tmp_path / idt
        write_csr_store(path, ip, ix, dv, nv, 16, 4, idt=idt)
        it = R.BatchIterator(path, R.LoaderConfig(16, 64, 32, 2), 0, staging="stream_pinned", output="csr")
        for b in it:
            mb = b.to_minibatch()
            eip, eix, edv = csr_gather(ip, ix, dv, mb.global_indices)
            assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
            assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
        assert it.counters().h2d_bytes >= it.counters().bytes_read
        it.close()


@pytest.mark.parametrize("vdt", ["f32", "i32"])
def test_counts_store_staging(tmp_path, vdt):
    """Procedural counts (BASELINE config 2's shape): integer values in [1, 64]
    stage as one byte per value (kD8Int8), f32 and i32 alike.  Batches bit-exact,
    normalize within 1e-6."""
    path = tmp_path / "s"
    R.synth_store(path, R.SynthConfig(n_obs=600, n_var=9000, layout="csr", value_dtype=vdt, seed=4, chunk_rows=64,
                                      chunks_per_shard=4, counts=True))
    ip, ix, dv = load_csr_store(path)
    for out, xf in (("csr", None), ("dense", None), ("dense", "normalize_log1p")):
        it = R.BatchIterator(path, R.LoaderConfig(64, 256, 100, 1), 0, staging="stream_pinned", output=out,
                             out_dtype="f32" if xf else "native", transform=xf)
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if out == "csr":
                mb = b.to_minibatch()
                assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
                assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
            elif xf is None:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, 9000).tobytes()
            else:
                want = normalize_log1p(to_dense(eip, eix, edv.astype(np.float32), 9000))
                np.testing.assert_allclose(b.data.cpu().numpy().astype(np.float64), want, rtol=1e-6, atol=0)
        c = it.counters()
        assert c.h2d_bytes < 0.45 * c.bytes_read
        it.close()


def test_two_iterators_share_one_store(crafted):
    """Two iterators over ONE stream_pinned DeviceStore, next() calls interleaved:
    they share the store's block-slot pool (slots released by one are reused by
    the other behind its release event) and, after close, the output-buffer
    pool.  Both streams stay bit-exact."""
    path, ip, ix, dv = crafted
    ds = R.DeviceStore(path, 0, "stream_pinned")
    for rnd in range(2):  # second round reuses the pooled output buffers
        its = [R.BatchIterator(ds, R.LoaderConfig(16, 96, 40, 3 + k), k + rnd, output=out)
               for k, out in enumerate(("csr", "dense"))]
        live = [True, True]
        while any(live):
            for k, it in enumerate(its):
                if not live[k]:
                    continue
                b = it.next()
                if b is None:
                    live[k] = False
                    continue
                g = b.global_indices_host
                eip, eix, edv = csr_gather(ip, ix, dv, g)
                if k == 0:
                    mb = b.to_minibatch()
                    assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
                    assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
                else:
                    assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, NV).tobytes()
        for it in its:
            it.close()
    ds.close()


def test_iterators_on_threads_share_one_store(crafted):
    """Many iterators may share one store (loader.hpp:55-57): four host threads
    each run a whole epoch over one stream_pinned DeviceStore concurrently."""
    import threading
    path, ip, ix, dv = crafted
    ds = R.DeviceStore(path, 0, "stream_pinned")
    errors = []

    def run(k):
        try:
            torch.cuda.set_device(0)
            it = R.BatchIterator(ds, R.LoaderConfig(16, 96, 40, 10 + k), k, output="csr")
            for b in it:
                mb = b.to_minibatch()
                eip, eix, edv = csr_gather(ip, ix, dv, mb.global_indices)
                assert (np.asarray(mb.block.indices, np.uint64) == eix).all()
                assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
            it.close()
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ds.close()
    assert not errors, errors


def _fused_store(tmp_path, values, seed=11):
    """Rows of 0, 1, 2 and 1,000 .. 4,081 entries (4,081 = the fused kernel's
    limit with an unaligned row start) over 6,000 columns: every gap <= 255, so
    every record stages as a delta record and the store qualifies for K3d."""
    rng = np.random.default_rng(seed)
    n, nv = 200, 6000
    nnz = rng.integers(1000, 4082, n)
    nnz[::17] = 4081
    nnz[3::29] = 0
    nnz[5::31] = 1
    nnz[7::37] = 2
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    def cols(k):
        if k == 2:  # a gap of exactly 255 (the delta limit)
            c = int(rng.integers(0, nv - 256))
            return np.array([c, c + 255])
        return np.sort(rng.choice(nv, k, replace=False))
    ix = np.concatenate([cols(k) for k in nnz]).astype(np.uint64)
    if values == "counts":    # integer counts in [0, 255] as f32 -> kD8Int8 (one byte per value)
        dv = rng.integers(0, 64, len(ix)).astype(np.float32)
        dv[::97] = 255.0
    elif values == "halves":  # k / 2 as f32: <= 8 significant bits, low 16 bits zero -> kD8Coded16
        dv = (rng.integers(1, 200, len(ix)) / 2.0).astype(np.float32)
    elif values == "i32_small":  # i32 counts in [0, 255] -> kD8Int8
        dv = rng.integers(0, 256, len(ix)).astype(np.int32)
    elif values == "i32":
        dv = rng.integers(-50, 5000, len(ix)).astype(np.int32)
    else:                      # random floats with top-byte escapes -> kD8Coded ("signed": some negative)
        dv = (rng.random(len(ix)) + 0.25).astype(np.float32)
        wide = rng.random(len(ix)) < 0.05
        mag = rng.standard_normal(wide.sum()) * 10.0 ** rng.integers(-8, 9, wide.sum())
        dv[wide] = (mag if values == "signed" else np.abs(mag)).astype(np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 64, 2, vdt="i32" if values.startswith("i32") else "f32")
    return tmp_path / "s", ip, ix, dv, nv


@pytest.mark.parametrize("values,raw", [("counts", False), ("halves", False), ("floats", False), ("floats", True),
                                        ("signed", False), ("i32", False), ("i32_small", False)])
@pytest.mark.parametrize("staging", ["stream_pinned", "resident_coded"])
def test_fused_densify_from_delta_records(tmp_path, monkeypatch, values, raw, staging):
    """K3d (densify straight from the staged delta records, no k_d8_decode):
    bit-exact f32 / bf16 / native dense batches and normalize+log1p within 1e-6,
    one kernel per batch; RFL_FUSED=0 (decode + idx16 densify) gives the same bytes."""
    if raw:
        monkeypatch.setenv("RFL_NARROW_VALUES", "0")  # delta records with raw 4-byte values (kD8Raw)
    path, ip, ix, dv, nv = _fused_store(tmp_path, values)
    ds = R.DeviceStore(R.StoreReader(path), 0, staging)
    assert ds.image_bytes()[1] > 0  # re-encoded staging image (delta records)
    # (normalize+log1p on non-negative values, where the north-star 1e-6 applies: with
    # negative entries x * T / sum can approach -1 and log1p is ill-conditioned there)
    outs = [("native", None), ("bf16", None)] + (
        [] if values in ("i32", "i32_small", "signed") else [("f32", "normalize_log1p")])
    for od, xf in outs:
        got, launched = {}, {}
        for fused in ("1", "0"):
            monkeypatch.setenv("RFL_FUSED", fused)
            it = R.BatchIterator(ds, R.LoaderConfig(64, 128, 96, 3), 0, output="dense", out_dtype=od, transform=xf)
            nb, batches = 0, []
            for b in it:
                g = b.global_indices_host
                eip, eix, edv = csr_gather(ip, ix, dv, g)
                dense = to_dense(eip, eix, edv, nv)
                if xf:
                    want = normalize_log1p(dense.astype(np.float32))
                    np.testing.assert_allclose(b.data.cpu().numpy().astype(np.float64), want, rtol=1e-6, atol=0)
                elif od == "bf16":
                    from oracle.oracle import f32_to_bf16_bits
                    gb = b.data.view(torch.int16).cpu().numpy().view(np.uint16)
                    assert (gb == f32_to_bf16_bits(dense.astype(np.float32))).all()
                else:
                    assert b.data.cpu().numpy().tobytes() == dense.tobytes()
                batches.append(b.data.view(torch.uint8).cpu().numpy().tobytes())
                nb += 1
            c = it.counters()
            if fused == "1" and staging == "resident_coded":
                assert c.kernels_launched == nb  # no decode launches, no staging copies
            elif fused == "1":  # + at most one staging pull kernel per batch
                assert nb <= c.kernels_launched <= 2 * nb
            else:
                assert c.kernels_launched > launched["1"]
            launched[fused] = c.kernels_launched
            it.close()
            got[fused] = batches
        assert got["1"] == got["0"]
    ds.close()


def test_fused_falls_back_for_long_rows(tmp_path):
    """A store with a row of 4,082 entries (one past K3d's limit) densifies through
    k_d8_decode + the idx16 densify instead, still bit-exact."""
    rng = np.random.default_rng(3)
    n, nv = 64, 6000
    nnz = rng.integers(100, 3000, n)
    nnz[10] = 4082
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate([np.sort(rng.choice(nv, k, replace=False)) for k in nnz]).astype(np.uint64)
    dv = rng.integers(1, 64, len(ix)).astype(np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 32, 2)
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(32, 64, 64, 0), 0, staging="stream_pinned", output="dense")
    nb = 0
    for b in it:
        eip, eix, edv = csr_gather(ip, ix, dv, b.global_indices_host)
        assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, nv).tobytes()
        nb += 1
    assert it.counters().kernels_launched > nb
    it.close()


@pytest.mark.parametrize("stage", ["pull", "ce"])
def test_staging_pull_many_blocks_per_group(tmp_path, monkeypatch, stage):
    """stream_pinned groups that fetch more than the pull kernel's 256 jobs per
    launch (f = 4 rows per block, 3 x 700-row batches per group: ~525 blocks), with
    records of odd sizes (not multiples of 16 B) and chunks smaller than blocks and
    larger; the staging pull (default) and the per-block copy-engine fallback
    (RFL_STAGE=ce) give the reference's CSR and dense batches bit for bit."""
    if stage == "ce":
        monkeypatch.setenv("RFL_STAGE", "ce")
    rng = np.random.default_rng(17)
    nv, n = 3001, 2100
    nnz = rng.integers(0, 40, n)
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate([np.sort(rng.choice(nv, k, replace=False)) for k in nnz]).astype(np.uint64)
    dv = rng.random(len(ix)).astype(np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 2, 64)  # 2-row chunks: a 4-row block spans 2 records
    ds = R.DeviceStore(R.StoreReader(tmp_path / "s"), 0, "stream_pinned")
    for output in ("csr", "dense"):
        it = R.BatchIterator(ds, R.LoaderConfig(4, 2048, 700, 5), 0, output=output, batches_per_launch=3)
        seen = 0
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if output == "csr":
                mb = b.to_minibatch()
                assert (mb.block.indptr == eip).all() and (mb.block.indices == eix).all()
                assert mb.block.data.tobytes() == edv.tobytes()
            else:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, nv).tobytes()
            seen += len(g)
        assert seen == n
        it.close()
    ds.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_int8_value_kind_edges(tmp_path, monkeypatch, fused):
    """kD8Int8 eligibility is exact: a record holding 255.0 / 0.0 stages one byte
    per value, while one holding -0.0, 256.0, 255.5 or a denormal keeps a coded
    value kind -- CSR and dense batches bit-exact either way (K3d and the
    decode path)."""
    monkeypatch.setenv("RFL_FUSED", fused)
    rng = np.random.default_rng(5)
    n, nv = 64 * 6, 700
    nnz = rng.integers(0, 60, n)
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate([np.sort(rng.choice(nv, k, replace=False)) for k in nnz]).astype(np.uint64)
    dv = rng.integers(0, 256, len(ix)).astype(np.float32)
    edges = [np.float32(-0.0), np.float32(256.0), np.float32(255.5), np.float32(1e-45), np.float32(255.0)]
    for r, e in enumerate(edges):  # one edge value in each of the first records (64 rows each)
        k0, k1 = int(ip[64 * r]), int(ip[64 * (r + 1)])
        if k1 > k0:
            dv[k0 + (k1 - k0) // 2] = e
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 64, 3)
    ds = R.DeviceStore(R.StoreReader(tmp_path / "s"), 0, "stream_pinned")
    for output in ("csr", "dense"):
        it = R.BatchIterator(ds, R.LoaderConfig(64, 256, 96, 2), 0, output=output)
        seen = 0
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if output == "csr":
                mb = b.to_minibatch()
                assert (mb.block.indptr == eip).all() and (mb.block.indices == eix).all()
                assert mb.block.data.tobytes() == edv.tobytes()
            else:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, nv).tobytes()
            seen += len(g)
        assert seen == n
        it.close()
    ds.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_packed_delta_widths(tmp_path, monkeypatch, fused):
    """Bit-packed deltas at every group width: runs of single-entry rows (16-entry
    groups of row starts only: width 0), consecutive columns (width 1), gaps of 255
    (width 8), a record of 3,000+ entries (skip table past 32 groups), nnz not a
    multiple of 16 -- CSR and dense batches bit-exact through the pinned image
    (K3d and the decode path)."""
    monkeypatch.setenv("RFL_FUSED", fused)
    rng = np.random.default_rng(23)
    nv = 6000
    rows = []
    for i in range(640):
        kind = (i // 32) % 5
        if kind == 0:
            rows.append(np.array([int(rng.integers(0, nv))]))                  # single entries
        elif kind == 1:
            s0 = int(rng.integers(0, nv - 100))
            rows.append(np.arange(s0, s0 + int(rng.integers(2, 90))))          # consecutive columns
        elif kind == 2:
            s0 = int(rng.integers(0, 300))
            rows.append(s0 + 255 * np.arange(int(rng.integers(2, 22))))        # gaps of 255
        elif kind == 3:
            rows.append(np.sort(rng.choice(nv, int(rng.integers(150, 400)), replace=False)))
        else:
            rows.append(np.array([], dtype=np.int64))
    rows[100] = np.sort(rng.choice(nv, 3100, replace=False))                    # a long row (many groups)
    nnz = np.array([len(r) for r in rows])
    ip = np.zeros(len(rows) + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate(rows).astype(np.uint64)
    dv = (rng.random(len(ix)) + 0.5).astype(np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 64, 4)
    n = len(rows)
    ds = R.DeviceStore(R.StoreReader(tmp_path / "s"), 0, "stream_pinned")
    for output in ("csr", "dense"):
        it = R.BatchIterator(ds, R.LoaderConfig(64, 256, 100, 4), 0, output=output)
        seen = 0
        for b in it:
            g = b.global_indices_host
            eip, eix, edv = csr_gather(ip, ix, dv, g)
            if output == "csr":
                mb = b.to_minibatch()
                assert (mb.block.indptr == eip).all() and (mb.block.indices == eix).all()
                assert mb.block.data.tobytes() == edv.tobytes()
            else:
                assert b.data.cpu().numpy().tobytes() == to_dense(eip, eix, edv, nv).tobytes()
            seen += len(g)
        assert seen == n
        it.close()
    ds.close()
