"""GPU parity at the BASELINE bench shapes (the shapes bench.py and profiles/
report), pinned to the compiled reference through tests/golden/shapes.json
(tests/golden/make_golden_shapes.py): the inputs are regenerated with the
product synth (byte-identical to the generator the golden used) and every
batch / output file is compared by FNV-1a hash with the reference's.

* cfg1 (100k x 20k CSR, f=64 B=b=4096): the whole of epoch 0 -- CSR batches
  streamed from pinned host memory through the delta-coded staging image, and
  densified batches from the HBM-resident image;
* cfg2 (36k-gene counts, f=1024 B=16384 b=4096): CSR + densify at width 36,000,
  plus the fused normalize+log1p against the fp64 restatement (rtol 1e-6), also
  on rows holding more entries (4,097 .. 12,000) than the kernel keeps in
  registers;
* cfg3 (12,288-byte u8 rows, f=256 b=1024): raw and u8 -> bf16, every work unit
  of a row (12 x 1 KB per row) through the gather kernels;
* cfg4 (4 x 1024 one-hot u8, f=512 b=2048): raw, HBM-resident and staged as
  2-bit channel codes; the one-hot staging gate for widths that are not a
  multiple of 64 bytes;
* cfg5 (run_shuffle, 62,710 genes, 4,096-row output chunks): every output file
  byte-identical, with records larger than the 64 MB D2H piece;
* the reference's multi-range read_rows_csr vectors (golden.json) through the
  raw rfl_csr_gather kernel.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2604_01949_b200 as R
from paper_2604_01949_b200 import _lib as L
from oracle.oracle import (Orc, csr_gather, f32_to_bf16_bits, load_csr_store, load_dense_store, normalize_log1p,
                           to_dense, write_csr_store)

from conftest import fnv

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SHAPES = json.loads((Path(__file__).resolve().parent / "golden" / "shapes.json").read_text())


def _synth(path, s):
    cfg = R.SynthConfig(s["n_obs"], s["n_var"], s["layout"], s["value_dtype"], s.get("index_dtype", "u32"),
                        s.get("density", 0.1), s["seed"], s["chunk_rows"], s["cps"],
                        counts=s["gen"] == "counts", one_hot=s.get("one_hot", 0))
    R.synth_store(path, cfg)
    return path


@pytest.fixture(scope="module")
def stores(tmp_path_factory):
    d = tmp_path_factory.mktemp("shapes")
    return {k: _synth(d / k, SHAPES[k]) for k in ("cfg1", "cfg2", "cfg3", "cfg4")}


def _cfg(s, **kw):
    ld = s["loader"]
    return R.LoaderConfig(ld["f"], ld["B"], ld["b"], ld["seed"], **kw)


def _check_counters(it, s, staging):
    c = it.counters()
    assert c.blocks_fetched == s["blocks_fetched"] and c.peak_buffer_rows == s["peak_buffer_rows"]
    assert (c.read_ops, c.bytes_read, c.chunks_decoded) == (s["read_ops"], s["bytes_read"], s["chunks_decoded"])


@pytest.mark.parametrize("staging,output", [("stream_pinned", "csr"), ("resident", "dense"),
                                            ("stream_file", "csr")])
def test_cfg1_epoch_vs_reference(stores, staging, output):
    s = SHAPES["cfg1"]
    it = R.BatchIterator(stores["cfg1"], _cfg(s, prefetch_depth=4), s["loader"]["epoch"], staging=staging,
                         output=output)
    k = 0
    for b in it:
        m = b.to_minibatch()
        assert hex(fnv([m.global_indices])) == s["gidx_fnv"][k]
        if output == "csr":
            assert hex(fnv([m.block.indptr, m.block.indices, m.block.data])) == s["csr_fnv"][k]
        else:
            assert hex(fnv([m.block.values])) == s["dense_fnv"][k]
        k += 1
    assert k == len(s["rows"])
    _check_counters(it, s, staging)
    it.close()


@pytest.mark.parametrize("staging", ["stream_pinned", "resident", "stream_file", "resident_coded"])
def test_cfg2_counts_vs_reference(stores, staging):
    s = SHAPES["cfg2"]
    for output, key in (("csr", "csr_fnv"), ("dense", "dense_fnv")):
        it = R.BatchIterator(stores["cfg2"], _cfg(s, prefetch_depth=2), 0, staging=staging, output=output)
        got = []
        for b in it:
            m = b.to_minibatch()
            assert hex(fnv([m.global_indices])) == s["gidx_fnv"][len(got)]
            got.append(hex(fnv([m.block.indptr, m.block.indices, m.block.data] if output == "csr"
                               else [m.block.values])))
        assert got == s[key]
        _check_counters(it, s, staging)
        it.close()


def _normalize_expect(ip, ix, dv, g):
    eip, eix, edv = csr_gather(ip, ix, dv, g)
    nnz = np.diff(eip.astype(np.int64))
    cs = np.concatenate([[0.0], np.cumsum(edv.astype(np.float64))])
    tot = cs[eip[1:].astype(np.int64)] - cs[eip[:-1].astype(np.int64)]
    scale = np.repeat(np.where(tot != 0, 1e4 / tot, 0.0), nnz)
    return eip, eix, edv, nnz, np.log1p(edv.astype(np.float64) * scale)


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "resident_coded"])
def test_cfg2_normalize_log1p(stores, staging):
    """Fused library-size normalisation (fp64 row sums, T=1e4) + log1p at width 36,000."""
    s = SHAPES["cfg2"]
    ip, ix, dv = load_csr_store(stores["cfg2"])
    it = R.BatchIterator(stores["cfg2"], _cfg(s), 0, staging=staging, output="dense", transform="normalize_log1p")
    for b in it:
        g = b.global_indices_host
        eip, eix, edv, nnz, want = _normalize_expect(ip, ix, dv, g)
        rows = torch.from_numpy(np.repeat(np.arange(len(g)), nnz)).cuda()
        d = b.data
        got = d[rows, torch.from_numpy(eix.astype(np.int64)).cuda()].double().cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=0)  # north-star tolerance
        assert int((d != 0).sum()) == int((edv != 0).sum())


@pytest.mark.parametrize("out_dtype", ["f32", "bf16"])
def test_normalize_rows_longer_than_registers(tmp_path, out_dtype):
    """Rows with 4,097 .. 12,000 entries (more than the kernel's register-held
    first pass) next to short and empty rows, 36k genes."""
    rng = np.random.default_rng(5)
    n, nv = 96, 36_000
    nnz = rng.integers(0, 3000, n)
    nnz[::3] = rng.integers(4097, 12_000, len(nnz[::3]))
    nnz[5] = 0
    ip = np.zeros(n + 1, np.uint64)
    ip[1:] = np.cumsum(nnz)
    ix = np.concatenate([np.sort(rng.choice(nv, k, replace=False)) for k in nnz]).astype(np.uint64)
    dv = rng.integers(1, 64, len(ix)).astype(np.float32)
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 32, 4)
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(32, 96, 48, 2), 0, output="dense", out_dtype=out_dtype,
                         transform="normalize_log1p")
    seen = 0
    for b in it:
        exp = normalize_log1p(to_dense(*csr_gather(ip, ix, dv, b.global_indices_host), nv), 1e4)
        if out_dtype == "f32":
            np.testing.assert_allclose(b.data.double().cpu().numpy(), exp, rtol=1e-6, atol=0)
        else:
            got = b.data.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.int64)
            want = f32_to_bf16_bits(exp.astype(np.float32)).astype(np.int64)
            assert np.abs(got - want).max() <= 1  # one bf16 ulp of the correctly rounded value
            assert ((got == 0) == (want == 0)).all()
        seen += b.n_rows
    assert seen == n


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file"])
def test_cfg3_dense_u8_and_bf16_vs_reference(stores, staging):
    s = SHAPES["cfg3"]
    for out_dtype, key in (("native", "dense_fnv"), ("bf16", "bf16_fnv")):
        it = R.BatchIterator(stores["cfg3"], _cfg(s, prefetch_depth=2), 0, staging=staging, output="dense",
                             out_dtype=out_dtype)
        got = []
        for b in it:
            assert hex(fnv([b.global_indices_host])) == s["gidx_fnv"][len(got)]
            x = b.data.view(torch.int16) if out_dtype == "bf16" else b.data
            got.append(hex(fnv([x.cpu().numpy()])))
        assert got == s[key]
        _check_counters(it, s, staging)
        it.close()


@pytest.mark.parametrize("staging", ["resident", "stream_pinned", "stream_file", "resident_coded"])
def test_cfg4_one_hot_vs_reference(stores, staging):
    s = SHAPES["cfg4"]
    ds = R.DeviceStore(stores["cfg4"], 0, staging)
    it = R.BatchIterator(ds, _cfg(s, prefetch_depth=2), 0, output="dense")
    got = []
    for b in it:
        assert hex(fnv([b.global_indices_host])) == s["gidx_fnv"][len(got)]
        got.append(hex(fnv([b.data.cpu().numpy()])))
    assert got == s["dense_fnv"]
    _check_counters(it, s, staging)
    if staging == "stream_pinned":  # staged as 2-bit channel codes: 1/16 of the row bytes crossed PCIe
        c = it.counters()
        assert c.h2d_bytes < c.bytes_read / 8
    it.close()
    ds.close()


@pytest.mark.parametrize("n_var", [48, 4000, 4096 + 16, 256, 64, 8192])
def test_one_hot_staging_widths(tmp_path, n_var):
    """One-hot rows whose width is not a multiple of 64 bytes stage verbatim (the
    2-bit decode needs 16-B chunks inside one channel plane); multiples of 64 use
    the coded image, read straight by K4o (64: one code word per row, 8192: two
    work units per row).  Bit-exact either way."""
    R.synth_store(tmp_path / "s", R.SynthConfig(700, n_var, "dense", "u8", seed=9, chunk_rows=64,
                                                chunks_per_shard=4, one_hot=4))
    x = load_dense_store(tmp_path / "s")
    it = R.BatchIterator(tmp_path / "s", R.LoaderConfig(64, 256, 100, 1), 0, staging="stream_pinned")
    seen = 0
    for b in it:
        assert (b.data.cpu().numpy() == x[b.global_indices_host.astype(np.int64)]).all()
        seen += b.n_rows
    assert seen == 700
    c = it.counters()
    if n_var % 64 == 0:  # 2-bit codes (1/16 of the row bytes) + the 16-B row references
        assert c.h2d_bytes <= c.bytes_read * (1 / 16 + 16 / n_var) * 1.25
    else:
        assert c.h2d_bytes >= c.bytes_read


def test_cfg5_shuffle_62k_genes_vs_reference(tmp_path):
    """run_shuffle at the Tahoe gene count with 4,096-row output chunks: each
    output record (~65 MB) is larger than the 64 MB D2H piece, so records
    straddle pieces; every output file == the reference's."""
    s = SHAPES["cfg5"]
    sh = s["shuffle"]
    _synth(tmp_path / "in", s)
    plan = R.plan_shuffle(s["n_obs"], sh["c"], sh["m"], sh["seed"])
    st = R.run_shuffle([tmp_path / "in"], plan, tmp_path / "out",
                       R.ShuffleOutputConfig(sh["out_chunk_rows"], sh["out_cps"]))
    out = tmp_path / "out"
    files = sorted(p.relative_to(out).as_posix() for p in out.rglob("*") if p.is_file())
    assert {f: (out / f).stat().st_size for f in files} == s["sizes"]
    assert max(s["sizes"].values()) > 64 << 20
    assert {f: hex(Orc.fnv1a64(np.frombuffer((out / f).read_bytes(), np.uint8))) for f in files} == s["files"]
    assert st.rounds_executed == s["rounds"] and st.peak_resident_rows == s["peak_resident_rows"]


def test_read_rows_csr_golden_through_gather(golden, golden_stores):
    """The reference's uneven-slice concatenation (read_rows_csr, store.cpp:590-614:
    multi-range requests, ranges out of order and across chunks) == the raw
    rfl_csr_gather kernel over the same rows."""
    for case in golden["read_rows_csr"]:
        path = golden_stores[case["store"]]
        ds = R.DeviceStore(path, 0, "resident")
        m = ds.manifest()
        rows = np.concatenate([np.arange(a, b, dtype=np.uint64) for a, b in case["ranges"]])
        base, offs = ds.arena()
        refs = np.zeros((len(rows), 2), np.uint64)
        refs[:, 0] = offs[rows.astype(np.int64) // m.chunk_rows]
        refs[:, 1] = rows
        d_refs = torch.from_numpy(refs.view(np.int64)).cuda()
        isz = 4 if m.index_dtype == "u32" else 8
        vsz = {"f32": 4, "f64": 8, "i32": 4, "u8": 1}[m.value_dtype]
        n, nnz = len(rows), case["nnz"]
        out_ip = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        out_ix = torch.zeros(max(nnz, 1) * isz, dtype=torch.uint8, device="cuda")
        out_dv = torch.zeros(max(nnz, 1) * vsz, dtype=torch.uint8, device="cuda")
        desc = ds.arena_desc()
        L.check(L.lib().rfl_csr_gather(C.byref(desc), d_refs.data_ptr(), n, out_ip.data_ptr(), out_ix.data_ptr(),
                                       out_dv.data_ptr(), None, None))
        torch.cuda.synchronize()
        ip = out_ip.cpu().numpy().view(np.uint64)
        ix = out_ix.cpu().numpy()[:nnz * isz].view(np.uint32 if isz == 4 else np.uint64).astype(np.uint64)
        dv = out_dv.cpu().numpy()[:nnz * vsz]
        assert int(ip[-1]) == nnz
        assert hex(fnv([ip, ix, dv])) == case["fnv"], case
        ds.close()


@pytest.mark.parametrize("staging", ["resident_coded", "stream_pinned", "stream_file"])
def test_cfg2_procedural_source_vs_reference(staging):
    """The never-materialised record source bench.py uses for config 2 at 10M
    cells: the same generator config as the golden cfg2 store, addressed as
    "procedural:counts?...", gives the reference's batches."""
    s = SHAPES["cfg2"]
    spec = (f"procedural:counts?n_obs={s['n_obs']}&n_var={s['n_var']}&seed={s['seed']}&chunk_rows={s['chunk_rows']}"
            f"&chunks_per_shard={s['cps']}")
    it = R.BatchIterator(R.StoreReader(spec), _cfg(s, prefetch_depth=2), 0, staging=staging, output="csr")
    got = []
    for b in it:
        m = b.to_minibatch()
        assert hex(fnv([m.global_indices])) == s["gidx_fnv"][len(got)]
        got.append(hex(fnv([m.block.indptr, m.block.indices, m.block.data])))
    assert got == s["csr_fnv"]
    _check_counters(it, s, staging)
    it.close()


def test_loader_kernel_timing_counters(stores):
    """time_kernels=True: CUDA events around each batch's expansion and assembly
    kernels accumulate into the counters (bench.py's per-kernel roofline)."""
    s = SHAPES["cfg2"]
    it = R.BatchIterator(stores["cfg2"], _cfg(s), 0, staging="resident_coded", output="dense", time_kernels=True)
    n = sum(1 for _ in it)
    it.synchronize()
    c = it.counters()
    assert n == len(s["rows"]) and c.assembly_ms > 0 and c.decode_ms > 0
