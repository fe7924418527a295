"""Parity at BASELINE config 1's full size (100k cells x 20k genes, ~2k nnz/cell,
f=64, B=b=4096): whole epochs through the GPU loader, checked against the
oracle's schedule replay (riffle_oracle.c) and the numpy restatement of the
gather, with size-independent properties that are still bit-exact:

* every batch's global_indices equal the replay's, and the epoch covers every
  row exactly once;
* densify: every stored entry sits at [row, col] with its exact value and the
  row has exactly as many non-zeros as it stores, i.e. the dense batch
  equals to_dense (block.cpp:135-146) without materialising it on the host;
* CSR output (streamed from pinned host memory, through the delta-encoded
  staging image expanded on the GPU): indptr / indices / data byte-identical to the concatenation
  (CsrBlock::append_rows, block.cpp:92-108);
* normalize + log1p: the non-zeros within 1e-6 relative of the fp64 oracle.
"""
import numpy as np
import pytest
import torch

import paper_2604_01949_b200 as R
from oracle.oracle import Orc, csr_gather, load_csr_store

pytestmark = pytest.mark.gpu

N, NV, F, B, BATCH = 100_000, 20_000, 64, 4096, 4096


@pytest.fixture(scope="module")
def cfg1(tmp_path_factory):
    path = tmp_path_factory.mktemp("cfg1") / "store"
    R.synth_store(path, R.SynthConfig(n_obs=N, n_var=NV, layout="csr", value_dtype="f32", index_dtype="u32",
                                      density=0.1, seed=0, chunk_rows=64, chunks_per_shard=128))
    ip, ix, dv = load_csr_store(path)
    return path, ip, ix, dv


def _expect(ip, ix, dv, g):
    eip, eix, edv = csr_gather(ip, ix, dv, g)
    nnz = np.diff(eip.astype(np.int64))
    rows = torch.from_numpy(np.repeat(np.arange(len(g)), nnz)).cuda()
    return eip, eix, edv, nnz, rows


def _nonzeros_per_row(eip, edv):
    """Stored entries that are non-zero, per row (synth's column-0 identity channel
    holds the row id, so row 0 stores an explicit 0.0)."""
    c = np.concatenate([[0], np.cumsum(edv != 0)])
    return torch.from_numpy((c[eip[1:].astype(np.int64)] - c[eip[:-1].astype(np.int64)]).astype(np.int64))


def test_cfg1_full_epoch_densify(cfg1):
    path, ip, ix, dv = cfg1
    sched, _, _ = Orc.replay_epoch(N, F, B, BATCH, seed=0, epoch=0)
    it = R.BatchIterator(path, R.LoaderConfig(F, B, BATCH, 0), 0, device=0, staging="resident", output="dense")
    seen = np.zeros(N, np.int64)
    k = 0
    for batch in it:
        g = batch.global_indices_host
        assert (g == sched[k]).all()
        seen[g.astype(np.int64)] += 1
        eip, eix, edv, nnz, rows = _expect(ip, ix, dv, g)
        d = batch.data
        assert d.shape == (len(g), NV) and d.dtype == torch.float32
        cols = torch.from_numpy(eix.astype(np.int64)).cuda()
        assert torch.equal(d[rows, cols], torch.from_numpy(edv).cuda())
        assert torch.equal((d != 0).sum(1).cpu(), _nonzeros_per_row(eip, edv))
        k += 1
    assert k == len(sched) and (seen == 1).all()


def test_cfg1_full_epoch_csr_streamed(cfg1):
    path, ip, ix, dv = cfg1
    sched, _, _ = Orc.replay_epoch(N, F, B, BATCH, seed=0, epoch=1)
    it = R.BatchIterator(path, R.LoaderConfig(F, B, BATCH, 0, prefetch_depth=4), 1, device=0,
                         staging="stream_pinned", output="csr")
    k = 0
    for batch in it:
        mb = batch.to_minibatch()
        g = np.asarray(mb.global_indices, np.uint64)
        assert (g == sched[k]).all()
        eip, eix, edv = csr_gather(ip, ix, dv, g)
        assert (np.asarray(mb.block.indptr, np.uint64) == eip).all()
        assert (np.asarray(mb.block.indices, np.uint64) == eix.astype(np.uint64)).all()
        assert np.asarray(mb.block.data).tobytes() == edv.tobytes()
        k += 1
    assert k == len(sched)
    # the pinned staging image carried u8 column deltas (every in-row gap <= 255
    # in this store) and top-byte coded values: ~4.3 of every 8 record bytes per
    # entry crossed PCIe
    c = it.counters()
    assert 0.45 * c.bytes_read < c.h2d_bytes < 0.6 * c.bytes_read


def test_cfg1_normalize_log1p_full_rows(cfg1):
    path, ip, ix, dv = cfg1
    it = R.BatchIterator(path, R.LoaderConfig(F, B, BATCH, 3), 0, device=0, staging="resident", output="dense",
                         transform="normalize_log1p")
    for _, batch in zip(range(3), it):
        g = batch.global_indices_host
        eip, eix, edv, nnz, rows = _expect(ip, ix, dv, g)
        cs = np.concatenate([[0.0], np.cumsum(edv.astype(np.float64))])
        s = cs[eip[1:].astype(np.int64)] - cs[eip[:-1].astype(np.int64)]
        scale = np.repeat(np.where(s != 0, 1e4 / s, 0.0), nnz)
        want = np.log1p(edv.astype(np.float64) * scale)
        d = batch.data
        got = d[rows, torch.from_numpy(eix.astype(np.int64)).cuda()].double().cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=0)
        assert torch.equal((d != 0).sum(1).cpu(), _nonzeros_per_row(eip, edv))
