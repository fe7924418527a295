"""GPU pre-shuffle parity: the device writer's output store + provenance
sidecar are byte-identical to the reference run_shuffle (golden digests and
live oracle/_ref runs), including multi-member collections, chunks that
straddle rounds (out chunk_rows > m), index-dtype conversion and dense stores."""
import json
import os
from pathlib import Path

import numpy as np
import pytest

import paper_2604_01949_b200 as R
from oracle.oracle import Orc, Ref

pytestmark = pytest.mark.gpu


def digests(root: Path):
    return {p.relative_to(root).as_posix(): hex(Orc.fnv1a64(np.frombuffer(p.read_bytes(), np.uint8)))
            for p in sorted(root.rglob("*")) if p.is_file()}


def same_tree(a: Path, b: Path):
    fa = sorted(p.relative_to(a).as_posix() for p in a.rglob("*") if p.is_file())
    fb = sorted(p.relative_to(b).as_posix() for p in b.rglob("*") if p.is_file())
    assert fa == fb
    for f in fa:
        assert (a / f).read_bytes() == (b / f).read_bytes(), f


def test_golden_shuffles(golden, golden_stores, tmp_path):
    for case in golden["run_shuffle"]:
        out = tmp_path / f"gpu_{case['store']}"
        plan = R.plan_shuffle(golden["stores"][case["store"]]["n_obs"], case["c"], case["m"], case["seed"])
        st = R.run_shuffle([golden_stores[case["store"]]], plan, out,
                           R.ShuffleOutputConfig(case["out_chunk_rows"], case["out_cps"]))
        assert digests(out) == case["files"], case["store"]
        assert st.peak_resident_rows == case["peak_resident_rows"]
        assert st.rounds_executed == case["rounds"]


@pytest.mark.parametrize("c,m,ocr,ocps,seed", [(64, 512, 100, 4, 7), (7, 50, 333, 2, 1), (1, 40, 16, 3, 2),
                                               (500, 500, 64, 128, 3), (13, 13, 13, 1, 4)])
def test_live_reference_multi_member(tmp_path, c, m, ocr, ocps, seed):
    """Two members (identity columns), rounds crossing members, carried chunks."""
    a, b = tmp_path / "a", tmp_path / "b"
    R.synth_store(a, R.SynthConfig(700, 90, "csr", "f32", "u32", 0.1, 1, 32, 4))
    R.synth_store(b, R.SynthConfig(333, 90, "csr", "f32", "u32", 0.2, 2, 50, 2))
    Ref.run_shuffle([a, b], tmp_path / "ref", c, m, seed, ocr, ocps)
    plan = R.plan_shuffle(1033, c, m, seed)
    R.run_shuffle([a, b], plan, tmp_path / "gpu", R.ShuffleOutputConfig(ocr, ocps))
    same_tree(tmp_path / "ref", tmp_path / "gpu")


@pytest.mark.parametrize("layout,vdt,idt,out_idt", [("csr", "f64", "u64", "u32"), ("csr", "u8", "u32", "u64"),
                                                    ("dense", "f32", "u32", None), ("dense", "u8", "u32", None),
                                                    ("csr", "i32", "u32", None)])
def test_live_reference_dtypes(tmp_path, layout, vdt, idt, out_idt):
    R.synth_store(tmp_path / "in", R.SynthConfig(1500, 37, layout, vdt, idt, 0.15, 5, 64, 3))
    Ref.run_shuffle([tmp_path / "in"], tmp_path / "ref", 16, 200, 11, 77, 3, out_idt=out_idt)
    R.run_shuffle([tmp_path / "in"], R.plan_shuffle(1500, 16, 200, 11), tmp_path / "gpu",
                  R.ShuffleOutputConfig(77, 3, index_dtype=out_idt))
    same_tree(tmp_path / "ref", tmp_path / "gpu")


def test_shuffle_provenance_is_the_order(tmp_path):
    R.synth_store(tmp_path / "in", R.SynthConfig(5000, 20, "csr", "f32", "u32", 0.2, 0, 100, 8))
    R.run_shuffle([tmp_path / "in"], R.plan_shuffle(5000, 50, 1000, 3), tmp_path / "out",
                  R.ShuffleOutputConfig(256, 4))
    # column 0 carries the source row id (synth identity channel): read it back through the GPU loader
    it = R.BatchIterator(tmp_path / "out", R.LoaderConfig(256, 256, 256, 0), 0, output="csr")
    ids = {}
    for bt in it:
        mb = bt.to_minibatch()
        for k, g in enumerate(mb.global_indices):
            lo = int(mb.block.indptr[k])
            assert mb.block.indices[lo] == 0
            ids[int(g)] = int(mb.block.data[lo])
    order = R.shuffle_order(5000, 50, 1000, 3)
    assert [ids[o] for o in range(5000)] == order.tolist()


def _rank_shuffle(rank, world, inputs, total, out, c, m, seed, ocr, ocps, out_idt, a2a=None):
    import paper_2604_01949_b200 as R
    st = R.run_shuffle(inputs, R.plan_shuffle(total, c, m, seed), out,
                       R.ShuffleOutputConfig(ocr, ocps, index_dtype=out_idt), device=0, rank=rank, world=world,
                       a2a=a2a)
    assert st.a2a == (a2a or "ipc")  # auto on one GPU: every pair is "peer accessible" (same device)
    return st.rows_written


@pytest.mark.parametrize("world,c,m,ocr,ocps,layout,out_idt", [
    (2, 64, 512, 100, 2, "csr", None), (2, 7, 90, 333, 1, "csr", "u64"), (3, 16, 256, 40, 3, "csr", None),
    (2, 32, 300, 50, 2, "dense", None)])
def test_multi_rank_shuffle_byte_identical(tmp_path, world, c, m, ocr, ocps, layout, out_idt):
    """The multi-GPU data path (pack kernel writing into the owners' receive
    buffers through CUDA IPC peer pointers), with `world` processes sharing this
    box's GPU(s), gloo for the control plane: output == reference run_shuffle."""
    from test_multirank import _run
    a, b = tmp_path / "a", tmp_path / "b"
    R.synth_store(a, R.SynthConfig(1500, 60, layout, "f32", "u32", 0.1, 1, 32, 4))
    R.synth_store(b, R.SynthConfig(450, 60, layout, "f32", "u32", 0.2, 2, 50, 2))
    Ref.run_shuffle([a, b], tmp_path / "ref", c, m, 5, ocr, ocps, out_idt=out_idt)
    rows = _run(world, _rank_shuffle, [str(a), str(b)], 1950, str(tmp_path / "gpu"), c, m, 5, ocr, ocps, out_idt)
    assert sum(rows) == 1950
    same_tree(tmp_path / "ref", tmp_path / "gpu")


@pytest.mark.parametrize("world,layout", [(2, "csr"), (3, "csr"), (2, "dense")])
def test_multi_rank_shuffle_a2a_exchange(tmp_path, world, layout):
    """The all-to-all exchange variant (a2a="nccl": the pack kernel fills a local
    send buffer, one all_to_all_single per round moves the messages -- NCCL on a
    multi-GPU node, host-staged under gloo here): byte-identical output too."""
    from test_multirank import _run
    a, b = tmp_path / "a", tmp_path / "b"
    R.synth_store(a, R.SynthConfig(1500, 60, layout, "f32", "u32", 0.1, 1, 32, 4))
    R.synth_store(b, R.SynthConfig(450, 60, layout, "f32", "u32", 0.2, 2, 50, 2))
    Ref.run_shuffle([a, b], tmp_path / "ref", 16, 256, 5, 40, 3)
    rows = _run(world, _rank_shuffle, [str(a), str(b)], 1950, str(tmp_path / "gpu"), 16, 256, 5, 40, 3, None,
                "nccl")
    assert sum(rows) == 1950
    same_tree(tmp_path / "ref", tmp_path / "gpu")


def test_shuffle_errors(tmp_path):
    R.synth_store(tmp_path / "a", R.SynthConfig(100, 10, "csr", density=0.3, chunk_rows=10))
    R.synth_store(tmp_path / "d", R.SynthConfig(100, 10, "dense", chunk_rows=10))
    (tmp_path / "busy").mkdir()
    (tmp_path / "busy" / "x").write_text("x")
    plan = R.plan_shuffle(100, 10, 30, 0)
    with pytest.raises(R.InvalidArgument, match="not fresh"):
        R.run_shuffle([tmp_path / "a"], plan, tmp_path / "busy")
    with pytest.raises(R.InvalidArgument, match="empty collection"):
        R.run_shuffle([], plan, tmp_path / "o1")
    with pytest.raises(R.InvalidArgument, match="layout"):
        R.run_shuffle([tmp_path / "a", tmp_path / "d"], R.plan_shuffle(200, 10, 30, 0), tmp_path / "o2")


# ---- column reprojection (DatasetCollection joins, collection.cpp:28-82; preshuffle.cpp:95-134) ----
def set_var_names(path, names):
    """Give a store new var names (the shards do not depend on them)."""
    p = Path(path) / "manifest.json"
    m = json.loads(p.read_text())
    assert len(names) == m["n_var"]
    m["var_names"] = list(names)
    p.write_text(json.dumps(m, indent=2))


def _join_stores(tmp_path, layout, vdt, idt_a="u32", idt_b="u32"):
    """a: names v0..v89; b: 70 columns = a permuted subset of a's names plus
    names only b has; c: a's names in reverse order (same axis, not identity)."""
    rng = np.random.default_rng(3)
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    R.synth_store(a, R.SynthConfig(700, 90, layout, vdt, idt_a, 0.15, 1, 32, 4))
    R.synth_store(b, R.SynthConfig(333, 70, layout, vdt, idt_b, 0.3, 2, 50, 2))
    R.synth_store(c, R.SynthConfig(210, 90, layout, vdt, idt_a, 0.1, 3, 40, 2))
    shared = rng.permutation(90)[:55]
    names_b = [f"v{j}" for j in shared] + [f"b_only{j}" for j in range(15)]
    set_var_names(b, list(rng.permutation(names_b)))
    set_var_names(c, [f"v{j}" for j in reversed(range(90))])
    return [a, b, c], 1243


@pytest.mark.parametrize("layout,vdt,join", [("csr", "f32", "outer"), ("csr", "f32", "inner"),
                                             ("csr", "f64", "outer"), ("csr", "u8", "inner"),
                                             ("dense", "f32", "outer"), ("dense", "u8", "inner"),
                                             ("dense", "f64", "outer")])
def test_live_reference_reprojection(tmp_path, layout, vdt, join):
    """Members with differing var axes: GPU reprojection == reference run_shuffle, byte for byte."""
    ins, total = _join_stores(tmp_path, layout, vdt)
    Ref.run_shuffle(ins, tmp_path / "ref", 24, 300, 9, 100, 3, outer=(join == "outer"))
    R.run_shuffle(ins, R.plan_shuffle(total, 24, 300, 9), tmp_path / "gpu", R.ShuffleOutputConfig(100, 3), join=join)
    same_tree(tmp_path / "ref", tmp_path / "gpu")


@pytest.mark.parametrize("out_idt", [None, "u64"])
def test_live_reference_mixed_index_dtypes(tmp_path, out_idt):
    """Members with u32 and u64 indices (identity and remapped axes) are converted on the GPU."""
    ins, total = _join_stores(tmp_path, "csr", "f32", idt_a="u64", idt_b="u32")
    Ref.run_shuffle(ins, tmp_path / "ref", 16, 256, 4, 64, 2, out_idt=out_idt)
    R.run_shuffle(ins, R.plan_shuffle(total, 16, 256, 4), tmp_path / "gpu",
                  R.ShuffleOutputConfig(64, 2, index_dtype=out_idt))
    same_tree(tmp_path / "ref", tmp_path / "gpu")


def test_reprojection_duplicate_names_error(tmp_path):
    """Two member columns with one name map to one unified column: the reference
    rejects the emitted block (CsrBlock::validate); so does the GPU path, same message."""
    a, b = tmp_path / "a", tmp_path / "b"
    R.synth_store(a, R.SynthConfig(200, 20, "csr", "f32", "u32", 0.5, 1, 20, 4))
    R.synth_store(b, R.SynthConfig(100, 20, "csr", "f32", "u32", 0.5, 2, 20, 4))
    set_var_names(b, [f"v{j}" for j in range(19)] + ["v3"])
    with pytest.raises(Exception) as ref_err:
        Ref.run_shuffle([a, b], tmp_path / "ref", 10, 100, 1, 50, 2)
    with pytest.raises(R.InvalidArgument) as gpu_err:
        R.run_shuffle([a, b], R.plan_shuffle(300, 10, 100, 1), tmp_path / "gpu", R.ShuffleOutputConfig(50, 2))
    assert str(ref_err.value).split(": ", 1)[-1] in str(gpu_err.value)


@pytest.mark.parametrize("world,layout,join", [(2, "csr", "outer"), (3, "dense", "inner")])
def test_multi_rank_reprojection(tmp_path, world, layout, join):
    from test_multirank import _run
    ins, total = _join_stores(tmp_path, layout, "f32")
    Ref.run_shuffle(ins, tmp_path / "ref", 32, 300, 5, 50, 2, outer=(join == "outer"))
    rows = _run(world, _rank_shuffle_join, [str(p) for p in ins], total, str(tmp_path / "gpu"), 32, 300, 5, 50, 2,
                join)
    assert sum(rows) == total
    same_tree(tmp_path / "ref", tmp_path / "gpu")


def _rank_shuffle_join(rank, world, inputs, total, out, c, m, seed, ocr, ocps, join):
    import paper_2604_01949_b200 as R
    st = R.run_shuffle(inputs, R.plan_shuffle(total, c, m, seed), out, R.ShuffleOutputConfig(ocr, ocps),
                       device=0, rank=rank, world=world, join=join)
    return st.rows_written


@pytest.mark.parametrize("bad", ["order", "range", "indptr", "header"])
def test_shuffle_corrupt_input_raises_like_reference(tmp_path, bad):
    """Staged input records get decode_record's checks (host: header, length,
    indptr) and CsrBlock::validate's column checks (GPU): same CorruptStore text."""
    from oracle.oracle import write_csr_store
    rng = np.random.default_rng(1)
    rows, nv = 40, 30
    ip = np.zeros(rows + 1, np.uint64)
    cols = []
    for r in range(rows):
        c = np.sort(rng.choice(nv, 5, replace=False))
        cols.append(c)
        ip[r + 1] = ip[r] + 5
    ix = np.concatenate(cols).astype(np.uint64)
    dv = rng.random(len(ix)).astype(np.float32)
    if bad == "order":
        ix[5 * 17 + 2] = ix[5 * 17 + 1]
    elif bad == "range":
        ix[5 * 23] = 99
    write_csr_store(tmp_path / "s", ip, ix, dv, nv, 8, 2)
    if bad in ("indptr", "header"):
        shard = sorted((tmp_path / "s" / "shards").iterdir())[1]
        raw = bytearray(shard.read_bytes())
        if bad == "indptr":
            raw[12 + 12:12 + 16] = (7).to_bytes(4, "little")
        else:
            raw[4:12] = (41).to_bytes(8, "little")
        shard.write_bytes(bytes(raw))
    with pytest.raises(RuntimeError) as ref:
        Ref.run_shuffle([tmp_path / "s"], tmp_path / "ref", 4, 16, 3, 10, 2)
    with pytest.raises(R.CorruptStore) as ours:
        R.run_shuffle([tmp_path / "s"], R.plan_shuffle(rows, 4, 16, 3), tmp_path / "gpu", R.ShuffleOutputConfig(10, 2))
    assert str(ours.value) in str(ref.value)
