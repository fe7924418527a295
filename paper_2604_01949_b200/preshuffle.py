"""Pre-shuffle — host mirror of riffle's plan_shuffle / run_shuffle
(reference include/riffle/preshuffle.hpp:19-88, src/preshuffle.cpp:150-378)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


@dataclass
class ShufflePlan:
    """ShufflePlan (preshuffle.hpp:19-34)."""
    seed: int
    block_rows: int
    buffer_rows: int
    total_rows: int
    rounds: list = field(default_factory=list)

    def block_count(self) -> int:
        return (self.total_rows + self.block_rows - 1) // self.block_rows if self.block_rows else 0

    def block_range(self, block_id: int):
        s = block_id * self.block_rows
        return s, min(s + self.block_rows, self.total_rows)


def plan_shuffle(total_rows: int, block_rows: int, buffer_rows: int, seed: int) -> ShufflePlan:
    """plan_shuffle (preshuffle.cpp:150-181)."""
    nr = C.c_uint64()
    L.check(L.lib().rfl_plan_shuffle(total_rows, block_rows, buffer_rows, seed, C.byref(nr), None, None))
    nb = (total_rows + block_rows - 1) // block_rows
    lens = np.zeros(max(nr.value, 1), np.uint64)
    ids = np.zeros(max(nb, 1), np.uint64)
    L.check(L.lib().rfl_plan_shuffle(total_rows, block_rows, buffer_rows, seed, C.byref(nr), lens.ctypes.data,
                                     ids.ctypes.data))
    rounds, k = [], 0
    for r in range(nr.value):
        rounds.append(ids[k:k + int(lens[r])].tolist())
        k += int(lens[r])
    return ShufflePlan(seed, block_rows, buffer_rows, total_rows, rounds)


def shuffle_order(total_rows: int, block_rows: int, buffer_rows: int, seed: int) -> np.ndarray:
    """Global input row of every output row of run_shuffle (index-computable)."""
    out = np.zeros(max(total_rows, 1), np.uint64)
    L.check(L.lib().rfl_shuffle_order(total_rows, block_rows, buffer_rows, seed, out.ctypes.data))
    return out[:total_rows]


@dataclass
class RoundRoute:
    """Routing of one round across W ranks."""
    round: int
    out_rows: np.ndarray   # global output row of each row, in output order
    src_rows: np.ndarray   # global input row
    src_rank: np.ndarray   # rank that staged the row's block (block index in round mod W)
    dst_rank: np.ndarray   # owner of the output shard holding the row


def round_routes(total_rows, block_rows, buffer_rows, seed, out_chunk_rows, out_chunks_per_shard, world):
    """All rounds' routes (host logic of the multi-GPU pre-shuffle)."""
    plan = plan_shuffle(total_rows, block_rows, buffer_rows, seed)
    out = []
    for r in range(len(plan.rounds)):
        first, n = C.c_uint64(), C.c_uint64()
        args = (total_rows, block_rows, buffer_rows, seed, out_chunk_rows, out_chunks_per_shard, world, r)
        L.check(L.lib().rfl_shuffle_round_routes(*args, C.byref(first), C.byref(n), None, None, None))
        src = np.zeros(n.value, np.uint64)
        sr = np.zeros(n.value, np.uint32)
        dr = np.zeros(n.value, np.uint32)
        L.check(L.lib().rfl_shuffle_round_routes(*args, C.byref(first), C.byref(n), src.ctypes.data, sr.ctypes.data,
                                                 dr.ctypes.data))
        out.append(RoundRoute(r, first.value + np.arange(n.value, dtype=np.uint64), src, sr.astype(np.int64),
                              dr.astype(np.int64)))
    return out


@dataclass
class ShuffleOutputConfig:
    """ShuffleOutputConfig (preshuffle.hpp:44-50)."""
    chunk_rows: int = 1024
    chunks_per_shard: int = 128
    codec: str = "none"
    index_dtype: str | None = None


@dataclass
class ShuffleRunStats:
    """ShuffleRunStats (preshuffle.hpp:69-77) + device counters."""
    peak_resident_rows: int = 0
    rows_written: int = 0
    rounds_executed: int = 0
    input_bytes_read: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    gpu_ms: float = 0.0
    send_ms: float = 0.0        # multi-GPU: send-side pack kernels (peer stores in "ipc" mode)
    peer_bytes: int = 0         # multi-GPU: message bytes addressed to other ranks
    exchange_s: float = 0.0     # multi-GPU: wall time of the exchange phase (send .. all peers landed)
    a2a: str = ""               # multi-GPU exchange: "ipc" (fused peer stores) or "nccl" (all-to-all)


def _stats(st) -> ShuffleRunStats:
    return ShuffleRunStats(st.peak_resident_rows, st.rows_written, st.rounds_executed, st.input_bytes_read,
                           st.h2d_bytes, st.d2h_bytes, st.gpu_ms, st.send_ms, st.peer_bytes)


def run_shuffle(inputs, plan: ShufflePlan, out_path, out_config: ShuffleOutputConfig | None = None, *,
                device: int = 0, join: str = "outer", rank: int = 0, world: int = 1, group=None,
                a2a: str | None = None) -> ShuffleRunStats:
    """run_shuffle (preshuffle.cpp:185-378) with the round gather/permute/pack on the GPU.

    `inputs` is the ordered list of member store paths (DatasetCollection order).
    world > 1: call on every rank (one process per GPU) with an initialised
    torch.distributed group for the control plane; row payloads move between
    GPUs through peer memory, written by the pack kernel (a2a="ipc"), or as one
    NCCL all-to-all per round (a2a="nccl"); default (None / RFL_A2A=auto): ipc
    when every pair of ranks' GPUs can access each other's memory, else nccl
    (see _run_ranks)."""
    oc = out_config or ShuffleOutputConfig()
    if oc.codec not in ("none", "deflate"):
        raise L.InvalidArgument(f"unknown codec {oc.codec!r}")
    if inputs:
        from .store import StoreReader
        held = sum(StoreReader(p).manifest().n_obs for p in inputs)
        if plan.total_rows != held:  # preshuffle.cpp:191-194
            raise L.InvalidArgument(f"run_shuffle: plan covers {plan.total_rows} rows, collection holds {held}")
    paths = [str(p).encode() for p in inputs]
    arr = (C.c_char_p * len(paths))(*paths)
    cfg = L.rfl_shuffle_config(plan.block_rows, plan.buffer_rows, plan.seed, oc.chunk_rows, oc.chunks_per_shard,
                               -1 if oc.index_dtype is None else {"u32": 0, "u64": 1}[oc.index_dtype], device,
                               int(join == "outer"), rank, world, int(oc.codec == "deflate"))
    if world > 1:
        return _run_ranks(arr, len(paths), str(out_path), cfg, device, rank, world, group, a2a)
    st = L.rfl_shuffle_stats()
    L.check(L.lib().rfl_run_shuffle(arr, len(paths), str(out_path).encode(), C.byref(cfg), C.byref(st)))
    return _stats(st)


def _a16(x: int) -> int:
    return (x + 15) // 16 * 16


def _ctl_device(group):
    import torch
    import torch.distributed as dist
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else \
        torch.device("cpu")


def _all_gather_i64(vals, world, group):
    """All-gather of a small int64 vector per rank (one collective; tensors, not pickles)."""
    import torch
    import torch.distributed as dist
    dev = _ctl_device(group)
    t = torch.tensor(vals, dtype=torch.int64, device=dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out])


def _ipc_capable(device, rank, world, group) -> bool:
    """Every pair of ranks on one host, each pair of their GPUs peer-accessible
    (cudaDeviceCanAccessPeer), agreed by all ranks."""
    import socket
    host = int.from_bytes(socket.gethostname().encode()[:8].ljust(8, b"\0"), "little") & ((1 << 63) - 1)
    info = _all_gather_i64([host, device], world, group)
    ok = 1
    for p in range(world):
        if int(info[p, 0]) != host:
            ok = 0
            break
        flag = C.c_int()
        if L.lib().rfl_device_can_access_peer(device, int(info[p, 1]), C.byref(flag)) != L.OK or not flag.value:
            ok = 0
            break
    return bool(_all_gather_i64([ok], world, group).min())


def _run_ranks(arr, n_in, out_path, cfg, device, rank, world, group, a2a=None) -> ShuffleRunStats:
    """One rank of the multi-GPU pre-shuffle.

    Data plane: block b of round r is staged by rank b mod W; each output row
    goes to the owner of its shard (s mod W).
      a2a="ipc":  the K5 pack kernel of the source rank encodes the rows for
                  owner d as one CSR record and stores it directly into d's
                  receive buffer through CUDA IPC peer pointers (NVLink P2P on a
                  multi-GPU node) -- gather and exchange are one kernel pass.
      a2a="nccl": the pack kernel writes each owner's record into a local send
                  buffer and one all-to-all(v) per round moves them
                  (torch.distributed all_to_all_single = grouped ncclSend/ncclRecv
                  under the nccl backend; staged through host memory under gloo).
    Control plane (torch.distributed, any backend): per round one all-gather of
    a small int64 vector (message sizes, receive-buffer version, IPC handle)."""
    import os
    import time

    import torch
    import torch.distributed as dist

    from .loader import cuda_tensor
    lib = L.lib()
    h = L.vp()
    nr = C.c_uint64()
    mode = a2a or os.environ.get("RFL_A2A", "auto")
    if mode == "auto":
        mode = "ipc" if _ipc_capable(device, rank, world, group) else "nccl"
    if mode not in ("ipc", "nccl"):
        raise L.InvalidArgument(f"unknown a2a mode {mode!r}")
    nccl = dist.get_backend(group) == "nccl"

    def create():
        L.check(lib.rfl_pshuf_create(arr, n_in, out_path.encode(), C.byref(cfg), C.byref(h), C.byref(nr)))

    if rank == 0:  # the fresh-output check runs before any rank creates directories
        create()
    dist.barrier(group=group)
    if rank != 0:
        create()
    peers = {}  # rank -> (version, device pointer)
    version = 0
    sbuf = None
    exchange_s = 0.0
    ptr, changed = L.vp(), C.c_int()
    handle = (C.c_ubyte * 64)()
    cap, hv = 0, []
    seen_vers = None  # receive-buffer versions of the last round (IPC opens are agreed when they change)
    try:
        if mode == "ipc":  # a first receive buffer, so every round's gather carries a valid handle
            L.check(lib.rfl_pshuf_recv_buffer(h, 16, C.byref(ptr), handle, C.byref(changed)))
            version, cap = 1, 16
            hv = np.frombuffer(bytes(handle), np.int64).tolist()
        for r in range(nr.value):
            send = np.zeros(world, np.uint64)
            L.check(lib.rfl_pshuf_stage(h, r, send.ctypes.data))
            if mode == "ipc":
                # one all-gather per round: message sizes + every receive buffer's capacity,
                # version and IPC handle; a second one only when some buffer had to grow
                infos = _all_gather_i64(send.astype(np.int64).tolist() + [cap, version] + hv, world, group)
                mat = infos[:, :world].astype(np.uint64)  # [src, dst]
                needs = [sum(_a16(int(mat[s, p])) for s in range(world)) for p in range(world)]
                if any(needs[p] > int(infos[p, world]) for p in range(world)):
                    if needs[rank] > cap:
                        L.check(lib.rfl_pshuf_recv_buffer(h, needs[rank], C.byref(ptr), handle, C.byref(changed)))
                        version += changed.value
                        cap = needs[rank]
                        hv = np.frombuffer(bytes(handle), np.int64).tolist()
                    infos = np.concatenate([infos[:, :world + 1],
                                            _all_gather_i64([version] + hv, world, group)], axis=1)
                opened, err = False, None
                for p in range(world):
                    if p == rank:
                        continue
                    ver = int(infos[p, world + 1])
                    if p not in peers or peers[p][0] != ver:
                        opened = True
                        try:
                            if p in peers:
                                L.check(lib.rfl_ipc_close(peers[p][1], device))
                                del peers[p]
                            hb = infos[p, world + 2:].astype(np.int64).tobytes()
                            pp = L.vp()
                            L.check(lib.rfl_ipc_open((C.c_ubyte * 64).from_buffer_copy(hb), device, C.byref(pp)))
                            peers[p] = (ver, pp.value)
                        except L.RiffleError as e:  # (agreed below: no rank may run ahead into the exchange)
                            err = e
                            break
                # (decided from the gathered versions, identically on every rank)
                vers = [int(infos[p, world + 1]) for p in range(world)]
                if vers != seen_vers:
                    seen_vers = vers
                    ok = _all_gather_i64([0 if err is not None else 1, 1 if opened else 0], world, group)
                    if ok[:, 0].min() == 0:
                        raise L.CudaError(f"pre-shuffle round {r}: opening a peer receive buffer (CUDA IPC) failed on "
                                          f"rank(s) {[int(q) for q in np.nonzero(ok[:, 0] == 0)[0]]}"
                                          + (f": {err}" if err is not None else "") + "; RFL_A2A=nccl avoids peer mappings")
                dst = (L.vp * world)()
                for d in range(world):
                    base = ptr.value if d == rank else peers[d][1]
                    dst[d] = base + sum(_a16(int(mat[s, d])) for s in range(rank))
                t0 = time.perf_counter()
                L.check(lib.rfl_pshuf_send(h, r, dst))
                dist.barrier(group=group)  # every peer write of this round has landed
                exchange_s += time.perf_counter() - t0
            else:
                mat = _all_gather_i64(send.astype(np.int64).tolist(), world, group).astype(np.uint64)
                need = sum(_a16(int(mat[s, rank])) for s in range(world))
                L.check(lib.rfl_pshuf_recv_buffer(h, max(need, 16), C.byref(ptr), None, C.byref(changed)))
                in_splits = [_a16(int(mat[rank, d])) for d in range(world)]
                out_splits = [_a16(int(mat[s, rank])) for s in range(world)]
                total = sum(in_splits)
                if sbuf is None or sbuf.numel() < max(total, 16):
                    sbuf = torch.empty(max(total, 16) + max(total, 16) // 4, dtype=torch.uint8,
                                       device=f"cuda:{device}")
                dst = (L.vp * world)()
                o = 0
                for d in range(world):
                    dst[d] = sbuf.data_ptr() + o
                    o += in_splits[d]
                t0 = time.perf_counter()
                L.check(lib.rfl_pshuf_send(h, r, dst))  # pack into the send buffer (stream synchronised)
                rview = cuda_tensor(ptr.value, (max(need, 16),), np.uint8, device)[:need]
                try:
                    if nccl:  # grouped ncclSend/ncclRecv over NVLink
                        dist.all_to_all_single(rview, sbuf[:total], out_splits, in_splits, group=group)
                        torch.cuda.current_stream(device).synchronize()
                    else:  # gloo: through host memory
                        host_out = torch.empty(need, dtype=torch.uint8)
                        dist.all_to_all_single(host_out, sbuf[:total].cpu(), out_splits, in_splits, group=group)
                        rview.copy_(host_out)
                        torch.cuda.current_stream(device).synchronize()
                except (RuntimeError, dist.DistError) as e:  # DistBackendError & co. -> RFL_ENCCL's exception
                    raise L.NcclError(f"pre-shuffle round {r}: all-to-all exchange failed: {e}") from e
                exchange_s += time.perf_counter() - t0
            recv = np.ascontiguousarray(mat[:, rank])
            L.check(lib.rfl_pshuf_emit(h, r, recv.ctypes.data))
            if mode == "ipc":
                dist.barrier(group=group)  # receive buffers are free again (peers write them next round)
        st = L.rfl_shuffle_stats()
        if rank != 0:
            L.check(lib.rfl_pshuf_finish(h, C.byref(st)))
        dist.barrier(group=group)
        if rank == 0:  # manifest.json + provenance/meta.json once every shard is on disk
            L.check(lib.rfl_pshuf_finish(h, C.byref(st)))
        dist.barrier(group=group)
        out = _stats(st)
        out.exchange_s = exchange_s
        out.a2a = mode
        return out
    finally:
        for _, (ver, p) in peers.items():
            lib.rfl_ipc_close(p, device)
        lib.rfl_pshuf_destroy(h)
