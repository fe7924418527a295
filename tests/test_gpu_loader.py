"""GPU parity: the sm_100a batch assembly path (through the C-ABI) against the
CPU oracle — the compiled reference's batches (golden hashes + live Ref calls)
and the numpy restatement.  Bit-exact for indices/indptr/permutations/raw
values; the fused normalize+log1p within 1e-6 relative (fp32 output), and
within one bf16 ulp of the correctly rounded oracle (bf16 output)."""
import ctypes as C

import numpy as np
import pytest

import paper_2604_01949_b200 as R
from paper_2604_01949_b200 import _lib as L
from oracle.oracle import (Ref, csr_gather, f32_to_bf16_bits, load_csr_store, load_dense_store, normalize_log1p,
                           read_manifest, to_dense, u8_to_bf16_bits, write_csr_store)

from conftest import fnv

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cfg(ld, **kw):
    return R.LoaderConfig(ld["f"], ld["B"], ld["b"], ld["seed"], drop_last=ld["drop_last"], **kw)


@pytest.fixture(scope="module")
def dstores(golden_stores):
    return {(n, s): R.DeviceStore(p, 0, s) for n, p in golden_stores.items()
            for s in ("resident", "stream_pinned", "stream_file")}


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
def test_csr_batches_bit_exact(golden, golden_stores, staging):
    """K2 csr_gather == reference MiniBatch (indptr, u64-widened indices, data, global_indices).
    A fresh DeviceStore per iterator, as the golden run used a fresh StoreReader
    (its first footer loads count into bytes_read)."""
    for ld in golden["loaders"]:
        if golden["stores"][ld["store"]]["layout"] != "csr":
            continue
        it = R.BatchIterator(R.DeviceStore(golden_stores[ld["store"]], 0, staging), _cfg(ld), ld["epoch"],
                             output="csr")
        got = [b.to_minibatch() for b in it]
        assert it.next() is None
        assert [m.global_indices.tolist() for m in got] == ld["gidx"]
        assert [hex(fnv([m.block.indptr, m.block.indices, m.block.data])) for m in got] == ld["csr_fnv"]
        c = it.counters()
        assert c.blocks_fetched == ld["blocks_fetched"] and c.peak_buffer_rows == ld["peak_buffer_rows"]
        # the reference's IoStats for the same fetches, in every staging mode (footer loads included)
        assert (c.read_ops, c.bytes_read, c.chunks_decoded) == (ld["read_ops"], ld["bytes_read"],
                                                                ld["chunks_decoded"])


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
def test_densify_bit_exact(golden, dstores, staging):
    """K3 densify == reference to_dense of each MiniBatch (block.cpp:135-146)."""
    for ld in golden["loaders"]:
        st = golden["stores"][ld["store"]]
        it = R.BatchIterator(dstores[(ld["store"], staging)], _cfg(ld), ld["epoch"], output="dense")
        got = [b.to_minibatch() for b in it]
        assert [m.global_indices.tolist() for m in got] == ld["gidx"]
        assert [hex(fnv([m.block.values])) for m in got] == ld["dense_fnv"], ld["store"]
        assert all(m.block.values.shape == (len(g), st["n_var"]) for m, g in zip(got, ld["gidx"]))


def test_live_reference_iterator(golden_stores):
    """Direct comparison with the reference BatchIterator on a fresh config."""
    path = golden_stores["csr_unaligned"]
    ref = list(Ref.iterate(path, 33, 150, 61, seed=12, epoch=4, want="csr,to_dense"))
    it = R.BatchIterator(path, R.LoaderConfig(33, 150, 61, 12), 4, output="csr")
    for r, b in zip(ref, it):
        m = b.to_minibatch()
        assert (m.global_indices == r["gidx"]).all()
        assert (m.block.indptr == r["indptr"]).all() and (m.block.indices == r["indices"]).all()
        assert m.block.data.tobytes() == r["data"].tobytes()
    it2 = R.BatchIterator(path, R.LoaderConfig(33, 150, 61, 12), 4, output="dense")
    for r, b in zip(ref, it2):
        assert b.to_minibatch().block.values.tobytes() == r["to_dense"].tobytes()


@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_normalize_log1p(golden_stores, out_dtype):
    """Fused library-size normalisation + log1p vs the fp64 numpy restatement."""
    path = golden_stores["csr_small"]
    ip, ix, dv = load_csr_store(path)
    n_var = read_manifest(path)["n_var"]
    it = R.BatchIterator(path, R.LoaderConfig(64, 512, 200, 3), 1, output="dense", out_dtype=out_dtype,
                         transform="normalize_log1p", target_sum=1e4)
    n = 0
    for b in it:
        g = b.global_indices_host
        exp = normalize_log1p(to_dense(*csr_gather(ip, ix, dv, g), n_var), 1e4)
        if out_dtype == "f32":
            got = b.data.float().cpu().numpy().astype(np.float64)
            # tolerance stated by the north star: 1e-6 relative
            np.testing.assert_allclose(got, exp, rtol=1e-6, atol=0)
        else:
            got = b.data.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.int64)
            want = f32_to_bf16_bits(exp.astype(np.float32)).astype(np.int64)
            assert np.abs(got - want).max() <= 1  # one bf16 ulp (sign-free, positive values)
            assert ((got == 0) == (want == 0)).all()
        n += len(g)
    assert n == 3000


def test_bf16_cast_dense_u8(golden_stores):
    """K4 dense gather with u8 -> bf16 cast: exact."""
    path = golden_stores["dense_u8"]
    X = load_dense_store(path)
    it = R.BatchIterator(path, R.LoaderConfig(256, 1024, 128, 0), 0, output="dense", out_dtype="bf16")
    for b in it:
        got = b.data.view(torch.int16).cpu().numpy().view(np.uint16)
        assert (got == u8_to_bf16_bits(X[b.global_indices_host.astype(np.int64)])).all()


def test_csr_f32_to_bf16_densify(golden_stores):
    path = golden_stores["csr_small"]
    ip, ix, dv = load_csr_store(path)
    it = R.BatchIterator(path, R.LoaderConfig(64, 512, 256, 0), 0, output="dense", out_dtype="bf16")
    for b in it:
        exp = to_dense(*csr_gather(ip, ix, dv, b.global_indices_host), 400)
        got = b.data.view(torch.int16).cpu().numpy().view(np.uint16)
        assert (got == f32_to_bf16_bits(exp)).all()


def _arena_refs(ds, gidx):
    base, offs = ds.arena()
    m = ds.manifest()
    refs = np.zeros((len(gidx), 2), np.uint64)
    refs[:, 0] = offs[np.asarray(gidx, np.int64) // m.chunk_rows]
    refs[:, 1] = gidx
    return torch.from_numpy(refs.view(np.int64)).cuda()


def test_raw_kernels_random_rows(golden_stores):
    """rfl_csr_gather / rfl_csr_densify on arbitrary row lists (repeats, any order)."""
    rng = np.random.default_rng(0)
    for name in ("csr_small", "csr_unaligned", "csr_u64_f64"):
        path = golden_stores[name]
        m = read_manifest(path)
        ip, ix, dv = load_csr_store(path)
        ds = R.DeviceStore(path, 0, "resident")
        desc = ds.arena_desc()
        for n in (1, 7, 300, 2049):
            g = rng.integers(0, m["n_obs"], n).astype(np.uint64)
            refs = _arena_refs(ds, g)
            ei, ex, ed = csr_gather(ip, ix, dv, g)
            out_ip = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
            isz = 4 if m["index_dtype"] == "u32" else 8
            out_ix = torch.zeros(max(len(ex), 1) * isz, dtype=torch.uint8, device="cuda")
            out_dv = torch.zeros(max(len(ed), 1) * ed.itemsize, dtype=torch.uint8, device="cuda")
            out_g = torch.zeros(n, dtype=torch.int64, device="cuda")
            L.check(L.lib().rfl_csr_gather(C.byref(desc), refs.data_ptr(), n, out_ip.data_ptr(), out_ix.data_ptr(),
                                           out_dv.data_ptr(), out_g.data_ptr(), None))
            torch.cuda.synchronize()
            assert (out_ip.cpu().numpy().view(np.uint64) == ei).all()
            gx = out_ix.cpu().numpy()[:len(ex) * isz].view(np.uint32 if isz == 4 else np.uint64)
            assert (gx.astype(np.uint64) == ex).all()
            assert out_dv.cpu().numpy()[:ed.nbytes].tobytes() == ed.tobytes()
            assert (out_g.cpu().numpy().view(np.uint64) == g).all()
            # host-planned indptr (no device scan), at a nonzero base entry
            base = 5
            pre = torch.from_numpy((ei.astype(np.int64) + base)).cuda()
            out_ix2 = torch.zeros_like(out_ix)
            out_dv2 = torch.zeros_like(out_dv)
            out_g2 = torch.zeros_like(out_g)
            L.check(L.lib().rfl_csr_gather_prefixed(C.byref(desc), refs.data_ptr(), n, pre.data_ptr(),
                                                    out_ix2.data_ptr(), out_dv2.data_ptr(), out_g2.data_ptr(), None))
            torch.cuda.synchronize()
            assert torch.equal(out_ix2, out_ix) and torch.equal(out_dv2, out_dv) and torch.equal(out_g2, out_g)
            dense = torch.zeros(n * m["n_var"] * ed.itemsize, dtype=torch.uint8, device="cuda")
            L.check(L.lib().rfl_csr_densify(C.byref(desc), refs.data_ptr(), n, L.NATIVE, L.XF_NONE, 0.0,
                                            dense.data_ptr(), None, None))
            torch.cuda.synchronize()
            assert dense.cpu().numpy().tobytes() == to_dense(ei, ex, ed, m["n_var"]).tobytes()


@pytest.mark.parametrize("n_var,vdt,od", [(30000, "f32", "native"), (60001, "f32", "bf16"), (5, "f32", "native"),
                                          (26000, "f64", "f32")])
def test_densify_tiles_and_unaligned(tmp_path, n_var, vdt, od):
    """Multi-tile rows (> 100 KB of output) and rows whose byte size is not a
    multiple of 16 (generic store path), plus empty rows."""
    rng = np.random.default_rng(n_var)
    n = 150
    nnz = np.minimum(rng.integers(0, 400, n), n_var)
    nnz[::7] = 0
    nnz[3] = min(n_var, 5000)
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate([np.sort(rng.choice(n_var, k, replace=False)) for k in nnz]).astype(np.uint64)
    dv = (rng.random(len(ix)) + 0.5).astype(np.float32 if vdt == "f32" else np.float64)
    write_csr_store(tmp_path / "s", ip, ix, dv, n_var, 16, 4, "u32", vdt)
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(16, 64, 50, 1), 0, output="dense", out_dtype=od)
    seen = 0
    for b in it:
        exp = to_dense(*csr_gather(ip, ix, dv, b.global_indices_host), n_var)
        if od == "bf16":
            got = b.data.view(torch.int16).cpu().numpy().view(np.uint16)
            assert (got == f32_to_bf16_bits(exp.astype(np.float32))).all()
        elif od == "f32":
            assert (b.data.cpu().numpy() == exp.astype(np.float32)).all()
        else:
            assert b.data.cpu().numpy().tobytes() == exp.tobytes()
        seen += b.n_rows
    assert seen == n


def test_empty_rows_and_edges(tmp_path):
    ip = np.array([0, 0, 3, 3, 5, 5, 5], np.uint64)
    ix = np.array([1, 4, 9, 0, 2], np.uint64)
    dv = np.arange(1, 6, dtype=np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, 10, 2, 2)
    for f, B, b, dl in [(2, 4, 3, False), (1, 6, 6, False), (6, 6, 4, True), (3, 3, 1, False)]:
        ref = list(Ref.iterate(tmp_path / "s", f, B, b, drop_last=dl, want="csr,to_dense"))
        for out in ("csr", "dense"):
            # batches are views into the loader's output ring: materialise each before the next
            got = [g.to_minibatch()
                   for g in R.BatchIterator(tmp_path / "s", R.LoaderConfig(f, B, b, drop_last=dl), 0, output=out)]
            assert len(got) == len(ref)
            for r, m in zip(ref, got):
                assert (m.global_indices == r["gidx"]).all()
                if out == "csr":
                    assert (m.block.indptr == r["indptr"]).all() and (m.block.indices == r["indices"]).all()
                else:
                    assert m.block.values.tobytes() == r["to_dense"].tobytes()


@pytest.mark.parametrize("staging", ["resident", "stream_pinned"])
@pytest.mark.parametrize("bad", ["range", "order"])
def test_corrupt_indices_raise_like_reference(tmp_path, staging, bad):
    """CsrBlock::validate (block.cpp:110-133) runs on the GPU: an out-of-range or
    non-increasing column index raises CorruptStore with the reference's message."""
    ip = np.array([0, 2, 5, 6, 8], np.uint64)
    ix = np.array([0, 3, 1, 4, 7, 2, 5, 9], np.uint64)
    if bad == "range":
        ix[6] = 500
    else:
        ix[7] = 5  # row 3: 5, 5
    dv = np.arange(8, dtype=np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, 10, 2, 2)
    with pytest.raises(RuntimeError) as ref:
        Ref.read_rows_csr(tmp_path / "s", [(0, 4)])
    with pytest.raises(R.CorruptStore) as ours:
        R.DeviceStore(tmp_path / "s", 0, staging)
    assert str(ours.value) in str(ref.value)


@pytest.mark.parametrize("bad", ["range", "order"])
def test_corrupt_indices_stream_file_raise_at_fetch(tmp_path, bad):
    """stream_file checks columns per fetch, as decode_record does (store.cpp:116-120):
    the fetch of the bad block raises IoError naming the block (loader.cpp:70-73)
    around the reference's CorruptStore text; earlier batches come out intact."""
    ip = np.arange(0, 8 * 2 + 1, 2, dtype=np.uint64)  # 8 rows x 2 entries, chunk_rows 2
    ix = np.tile(np.array([1, 3], np.uint64), 8)
    if bad == "range":
        ix[13] = 500   # row 6
    else:
        ix[13] = 1     # row 6: 1, 1
    dv = np.arange(16, dtype=np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, 10, 2, 2)
    with pytest.raises(RuntimeError) as ref:
        Ref.read_rows_csr(tmp_path / "s", [(6, 8)])
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(2, 2, 2, 0, prefetch_depth=2), 0, staging="stream_file")
    with pytest.raises(R.IoError) as ours:
        for _ in it:
            pass
    msg = str(ours.value)
    assert "fetch block [6, 8)" in msg
    assert msg.split("): ", 1)[1] in str(ref.value)


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
@pytest.mark.parametrize("bad", ["indptr", "tail", "header"])
def test_corrupt_indptr_raise_like_reference(tmp_path, staging, bad):
    """decode_record's header/length checks and validate's indptr checks
    (store.cpp:81-122, block.cpp:110-133): same CorruptStore text as the reference,
    prefixed "chunk q in shard s:" as process_shard wraps it (store.cpp:455-457)."""
    ip = np.array([0, 2, 5, 6, 8], np.uint64)
    ix = np.array([0, 3, 1, 4, 7, 2, 5, 9], np.uint64)
    dv = np.arange(8, dtype=np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, 10, 2, 2)
    shard = sorted((tmp_path / "s" / "shards").iterdir())[0]
    raw = bytearray(shard.read_bytes())
    if bad == "indptr":  # chunk 0 = rows 0,1: indptr [0, 2, 5] -> [0, 6, 5]
        raw[12 + 4:12 + 8] = (6).to_bytes(4, "little")
    elif bad == "tail":  # chunk 0 indptr[2] = 4 != nnz 5
        raw[12 + 8:12 + 12] = (4).to_bytes(4, "little")
    else:  # header declares 3 rows
        raw[0:4] = (3).to_bytes(4, "little")
    shard.write_bytes(bytes(raw))
    with pytest.raises(RuntimeError) as ref:
        Ref.read_rows_csr(tmp_path / "s", [(0, 4)])
    with pytest.raises(R.CorruptStore) as ours:
        R.DeviceStore(tmp_path / "s", 0, staging)
    assert str(ours.value) in str(ref.value)


def test_epoch_completeness_and_sharding(tmp_path):
    """SPEC acceptance 4 on the device: every row exactly once per epoch, per rank
    disjoint, union complete (SURVEY §8e sharding)."""
    R.synth_store(tmp_path / "s", R.SynthConfig(20000, 300, "csr", density=0.02, seed=3, chunk_rows=64))
    ds = R.DeviceStore(tmp_path / "s", 0, "stream_pinned")
    allg = []
    for k in range(3):
        it = R.BatchIterator(ds, R.LoaderConfig(64, 1024, 512, 5, rank=k, world=3), 2, output="csr")
        gs = [b.global_indices.cpu().numpy() for b in it]
        allg.append(np.concatenate(gs))
    assert sorted(np.concatenate(allg).tolist()) == list(range(20000))


def test_prefetch_depth_and_out_slots_invariance(golden_stores):
    path = golden_stores["csr_small"]
    outs = []
    for depth, slots, staging in [(0, 1, "resident"), (4, 3, "stream_file"), (1, 2, "stream_pinned")]:
        it = R.BatchIterator(path, R.LoaderConfig(32, 300, 100, 9, prefetch_depth=depth), 0, output="dense",
                             out_slots=slots, staging=staging)
        outs.append([hex(fnv([b.to_minibatch().block.values])) for b in it])
    assert outs[0] == outs[1] == outs[2]


def test_dense_store_paths(golden, dstores):
    """K4 dense gather (raw) for dense stores == reference DenseBuffer batches."""
    for ld in golden["loaders"]:
        if golden["stores"][ld["store"]]["layout"] != "dense":
            continue
        for staging in ("resident", "stream_file"):
            it = R.BatchIterator(dstores[(ld["store"], staging)], _cfg(ld), ld["epoch"])
            assert [hex(fnv([b.to_minibatch().block.values])) for b in it] == ld["dense_fnv"]


@pytest.mark.parametrize("depth,bypass", [(0, False), (3, True), (16, True)])
def test_stream_file_readahead(golden, golden_stores, depth, bypass):
    """stream_file staging through the BlockReader (read-ahead threads, O_DIRECT
    4 KiB-aligned spans with cache_bypass) == reference batches and counters."""
    for ld in golden["loaders"]:
        st = golden["stores"][ld["store"]]
        it = R.BatchIterator(golden_stores[ld["store"]], _cfg(ld, prefetch_depth=depth, cache_bypass=bypass),
                             ld["epoch"], output="dense", staging="stream_file")
        got = [b.to_minibatch() for b in it]
        assert [m.global_indices.tolist() for m in got] == ld["gidx"]
        assert [hex(fnv([m.block.values])) for m in got] == ld["dense_fnv"], ld["store"]
        c = it.counters()
        assert c.read_ops == ld["read_ops"] and c.chunks_decoded == ld["chunks_decoded"]
        assert st["n_var"] == got[0].block.values.shape[1]
        # bytes_read as the reference counts it with the same cache_bypass (aligned O_DIRECT spans)
        list(Ref.iterate(golden_stores[ld["store"]], ld["f"], ld["B"], ld["b"], seed=ld["seed"], epoch=ld["epoch"],
                         drop_last=ld["drop_last"], cache_bypass=bypass))
        assert c.bytes_read == Ref.last_counters["bytes_read"]


def test_stream_file_abandoned_and_io_error(tmp_path):
    """An iterator dropped mid-epoch stops its reader threads; a shard that
    vanishes under a running iterator surfaces as IoError naming the block
    (BlockPrefetcher::fetch_guarded, loader.cpp:61-74)."""
    R.synth_store(tmp_path / "s", R.SynthConfig(4000, 50, "csr", density=0.2, seed=2, chunk_rows=64,
                                                chunks_per_shard=4))
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(64, 512, 256, 1, prefetch_depth=8), 0, output="csr",
                         staging="stream_file")
    it.next()
    it.close()
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(64, 512, 256, 1, prefetch_depth=1), 0, output="csr",
                         staging="stream_file")
    it.next()
    for p in (tmp_path / "s" / "shards").iterdir():
        p.write_bytes(b"")  # truncate every shard: reads ahead of the consumer fail
    with pytest.raises(R.IoError, match=r"fetch block \[\d+, \d+\)"):
        for _ in range(100):
            if it.next() is None:
                break


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
@pytest.mark.parametrize("group", [3, 8])
def test_batches_per_launch(golden, golden_stores, staging, group):
    """batches_per_launch = k: k consecutive batches replayed (ahead, on the
    replay thread), staged, and assembled by one launch into one output slot,
    handed out one per next() or several per next_many(): the batch stream,
    CSR / dense contents and counters are the reference's."""
    for ld in golden["loaders"]:
        layout = golden["stores"][ld["store"]]["layout"]
        outs = ["csr", "dense"] if layout == "csr" else ["dense"]
        for out in outs:
            it = R.BatchIterator(R.DeviceStore(golden_stores[ld["store"]], 0, staging), _cfg(ld, prefetch_depth=2),
                                 ld["epoch"], output=out, batches_per_launch=group, out_slots=2)
            got = []
            while True:
                bs = it.next_many(2) if len(got) % 2 == 0 else [b for b in [it.next()] if b is not None]
                if not bs:
                    break
                got += [b.to_minibatch() for b in bs]
            assert it.next() is None and it.next_many(4) == []
            assert [m.global_indices.tolist() for m in got] == ld["gidx"]
            if out == "csr":
                assert [hex(fnv([m.block.indptr, m.block.indices, m.block.data])) for m in got] == ld["csr_fnv"]
            else:
                assert [hex(fnv([m.block.values])) for m in got] == ld["dense_fnv"]
            c = it.counters()
            assert c.blocks_fetched == ld["blocks_fetched"] and c.peak_buffer_rows == ld["peak_buffer_rows"]
            assert (c.read_ops, c.bytes_read, c.chunks_decoded) == (ld["read_ops"], ld["bytes_read"],
                                                                    ld["chunks_decoded"])
            it.close()


@pytest.mark.parametrize("n_var", [64, 4096, 8192])
def test_raw_onehot_gather_random_rows(tmp_path, n_var):
    """rfl_onehot_gather (K4o) over a resident_coded one-hot store's arena on
    arbitrary row lists (repeats, any order): bit-identical to rfl_dense_gather
    over the verbatim resident records and to the numpy row gather, u8 and bf16."""
    path = tmp_path / "oh"
    R.synth_store(path, R.SynthConfig(n_obs=1500, n_var=n_var, layout="dense", value_dtype="u8", seed=4,
                                      chunk_rows=128, chunks_per_shard=4, one_hot=4))
    x = load_dense_store(path).reshape(1500, n_var)
    coded = R.DeviceStore(path, 0, "resident_coded")
    plain = R.DeviceStore(path, 0, "resident")
    assert coded.image_bytes()[1] * 16 <= coded.image_bytes()[0] + 16 * 256 * 12
    rng = np.random.default_rng(1)
    for n in (1, 33, 1000, 4097):
        g = rng.integers(0, 1500, n).astype(np.uint64)
        for od, esz in ((L.NATIVE, 1), (L.BF16, 2)):
            outs = []
            for ds, fn in ((coded, L.lib().rfl_onehot_gather), (plain, L.lib().rfl_dense_gather)):
                desc = ds.arena_desc()
                refs = _arena_refs(ds, g)
                out = torch.full((n * n_var * esz,), 0x5A, dtype=torch.uint8, device="cuda")
                og = torch.zeros(n, dtype=torch.int64, device="cuda")
                L.check(fn(C.byref(desc), refs.data_ptr(), n, od, out.data_ptr(), og.data_ptr(), None))
                torch.cuda.synchronize()
                assert (og.cpu().numpy().view(np.uint64) == g).all()
                outs.append(out.cpu().numpy())
            want = x[g.astype(np.int64)]
            if od == L.BF16:
                want = u8_to_bf16_bits(want)
            assert outs[0].tobytes() == want.tobytes()
            assert outs[1].tobytes() == outs[0].tobytes()
    with pytest.raises(R.InvalidArgument):  # u8 rows cast to bf16 only, as rfl_dense_gather
        desc = coded.arena_desc()
        refs = _arena_refs(coded, np.zeros(1, np.uint64))
        out = torch.zeros(4 * n_var, dtype=torch.uint8, device="cuda")
        L.check(L.lib().rfl_onehot_gather(C.byref(desc), refs.data_ptr(), 1, L.F32, out.data_ptr(), None, None))
    coded.close()
    plain.close()


@pytest.mark.parametrize("staging", ["resident", "stream_pinned"])
def test_ids_to_host_async(golden, golden_stores, staging):
    """DeviceBatch.ids_to_host (rfl_ids_download_async): the queued D2H of each
    batch's device ids lands the reference's global row ids, in batch order,
    grouped launches included."""
    ld = golden["loaders"][0]
    it = R.BatchIterator(R.DeviceStore(golden_stores[ld["store"]], 0, staging), _cfg(ld), ld["epoch"],
                         batches_per_launch=3, out_slots=2, stream=torch.cuda.current_stream())
    host = torch.zeros(ld["b"] * 3, dtype=torch.int64).pin_memory()
    got = []
    while bs := it.next_many(3):
        off = 0
        for b in bs:
            b.ids_to_host(host.data_ptr() + 8 * off)
            off += b.n_rows
        torch.cuda.current_stream().synchronize()
        off = 0
        for b in bs:
            got.append(host[off:off + b.n_rows].tolist())
            off += b.n_rows
    assert got == ld["gidx"]
