"""Multi-process (gloo, world size 2 and 4, CPU) tests of the N>1 host logic:
the loader's per-rank partition (plan positions i == rank mod W,
sampler stream(2e+1).stream(rank)) and the pre-shuffle's routing (every output
row produced by exactly one owner, byte-level order identical to the
single-process run).  Ranks talk through torch.distributed exactly as bench.py
and the multi-GPU pre-shuffle do; only the device work is absent."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = [q.get() for _ in range(world)]
    errs = [r for r in res if isinstance(r, str)]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
    return res


def _entry(rank, world, port, fn, args, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put(fn(rank, world, *args))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


def _loader_rank(rank, world, n, f, B, b, seed, epoch):
    import paper_2604_01949_b200 as R
    from oracle.oracle import Orc
    cfg = R.LoaderConfig(f, B, b, seed, rank=rank, world=world)
    mine = np.concatenate([g for g in R.EpochSchedule(n, cfg, epoch)] or [np.zeros(0, np.uint64)])
    exp, _, _ = Orc.replay_epoch(n, f, B, b, seed, epoch, False, rank, world)
    assert (mine == np.concatenate(exp)).all()
    # gather every rank's ids and check the epoch partition
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(mine)]))
    mx = int(max(s.item() for s in sizes))
    buf = torch.full((mx,), -1, dtype=torch.int64)
    buf[:len(mine)] = torch.from_numpy(mine.astype(np.int64))
    outs = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(outs, buf)
    allids = torch.cat([o[:int(s.item())] for o, s in zip(outs, sizes)]).numpy()
    assert sorted(allids.tolist()) == list(range(n))
    return len(mine)


@pytest.mark.parametrize("world", [2, 4])
def test_loader_partition_gloo(world):
    counts = _run(world, _loader_rank, 30011, 64, 1024, 500, 3, 2)
    assert sum(counts) == 30011
    assert max(counts) - min(counts) <= 64 * 2  # plan positions are dealt round-robin


def _shuffle_route_rank(rank, world, total, c, m, seed, cr, cps):
    """Route every output row to its owner through a real gloo all_to_all and
    check each owner ends up with exactly its shards' rows, in output order."""
    import paper_2604_01949_b200 as R
    from oracle.oracle import Orc
    routes = R.preshuffle.round_routes(total, c, m, seed, cr, cps, world)
    got = {}
    for rt in routes:
        # this rank is the source of the rows whose block index in the round is == rank (mod W)
        send = [rt.src_rows[(rt.src_rank == rank) & (rt.dst_rank == d)] for d in range(world)]
        # exchange counts, then payload (the global input row ids stand in for the row bytes)
        cnt_in = torch.tensor([len(s) for s in send], dtype=torch.int64)
        cnt_out = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(cnt_out, cnt_in)
        payload_in = torch.from_numpy(np.concatenate(send).astype(np.int64)) if any(len(s) for s in send) \
            else torch.zeros(0, dtype=torch.int64)
        payload_out = torch.zeros(int(cnt_out.sum()), dtype=torch.int64)
        dist.all_to_all_single(payload_out, payload_in, cnt_out.tolist(), cnt_in.tolist())
        # owner side: merge the per-source messages back into output order
        recv = np.split(payload_out.numpy(), np.cumsum(cnt_out.numpy())[:-1])
        cursor = [0] * world
        mine = (rt.dst_rank == rank)
        for o, s in zip(rt.out_rows[mine], rt.src_rank[mine]):
            got[int(o)] = int(recv[s][cursor[s]])
            cursor[s] += 1
        assert cursor == [len(x) for x in recv]
    order = Orc.shuffle_order(total, c, m, seed)
    owned = [o for o in range(total) if (o // (cr * cps)) % world == rank]
    assert sorted(got) == owned
    assert all(got[o] == int(order[o]) for o in owned)
    return len(owned)


@pytest.mark.parametrize("world,total,c,m,cr,cps", [(2, 5000, 50, 1000, 128, 3), (2, 777, 7, 100, 333, 1),
                                                    (4, 4096, 64, 512, 64, 2)])
def test_preshuffle_routing_gloo(world, total, c, m, cr, cps):
    n = _run(world, _shuffle_route_rank, total, c, m, 11, cr, cps)
    assert sum(n) == total
