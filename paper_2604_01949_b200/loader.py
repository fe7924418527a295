"""GPU BatchIterator — host mirror of riffle's loader interface
(reference include/riffle/loader.hpp:12-81, src/loader.cpp:159-315).

Same names, argument meaning and error behaviour as the reference:
``LoaderConfig.validate`` raises InvalidArgument; ``next()`` returns None at
end of epoch (idempotently); a failed fetch raises IoError naming the block.
Batches live on the GPU (torch tensor views over the loader's output ring,
valid for ``out_slots`` further ``next()`` calls); ``DeviceBatch.to_minibatch``
materialises the reference's host MiniBatch (u64 indices) for parity checks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .store import DeviceStore, StoreReader

_NP = {L.F32: np.float32, L.F64: np.float64, L.I32: np.int32, L.U8: np.uint8, L.BF16: np.uint16}
_TYPESTR = {np.float32: "<f4", np.float64: "<f8", np.int32: "<i4", np.uint8: "|u1", np.uint16: "<u2",
            np.int64: "<i8", np.uint64: "<u8", np.uint32: "<u4"}
OUT_DTYPES = {"native": L.NATIVE, "f32": L.F32, "bf16": L.BF16}


@dataclass
class LoaderConfig:
    """LoaderConfig (loader.hpp:12-22) + rank/world (world=1 is the reference)."""
    fetch_block_rows: int = 1024
    buffer_capacity_rows: int = 16384
    batch_rows: int = 256
    seed: int = 0
    prefetch_depth: int = 0
    drop_last: bool = False
    cache_bypass: bool = False
    rank: int = 0
    world: int = 1
    even_batches: bool = False  # new: every rank stops after the smallest per-rank batch count (DDP-safe epochs)

    def _c(self) -> L.rfl_loader_config:
        return L.rfl_loader_config(self.fetch_block_rows, self.buffer_capacity_rows, self.batch_rows, self.seed,
                                   self.prefetch_depth, int(self.drop_last), int(self.cache_bypass), self.rank,
                                   self.world, int(self.even_batches))

    def validate(self) -> None:
        """loader.cpp:159-168."""
        L.check(L.lib().rfl_loader_config_validate(C.byref(self._c())))


@dataclass
class EpochPlan:
    blocks: list
    epoch_index: int = 0


def plan_epoch(n_obs: int, config: LoaderConfig, epoch_index: int) -> EpochPlan:
    """plan_epoch (loader.cpp:170-181)."""
    nb = (n_obs + config.fetch_block_rows - 1) // config.fetch_block_rows if config.fetch_block_rows else 0
    s = np.zeros(max(nb, 1), np.uint64)
    e = np.zeros(max(nb, 1), np.uint64)
    L.check(L.lib().rfl_plan_epoch(n_obs, C.byref(config._c()), epoch_index, s.ctypes.data, e.ctypes.data))
    return EpochPlan([(int(a), int(b)) for a, b in zip(s[:nb], e[:nb])], epoch_index)


class EpochSchedule:
    """Index-only replay of BatchIterator::next: the exact global_indices stream."""

    def __init__(self, n_obs: int, config: LoaderConfig, epoch_index: int = 0):
        self.config = config
        h = L.vp()
        L.check(L.lib().rfl_schedule_create(n_obs, C.byref(config._c()), epoch_index, C.byref(h)))
        self._h = h
        self._buf = np.zeros(config.batch_rows, np.uint64)

    def next(self):
        n = C.c_uint64()
        rc = L.check(L.lib().rfl_schedule_next(self._h, self._buf.ctypes.data, C.byref(n)))
        return None if rc == L.END else self._buf[: n.value].copy()

    def __iter__(self):
        while (g := self.next()) is not None:
            yield g

    def stats(self):
        p, b = C.c_uint64(), C.c_uint64()
        L.check(L.lib().rfl_schedule_stats(self._h, C.byref(p), C.byref(b)))
        return {"peak_buffer_rows": p.value, "blocks_fetched": b.value}

    def __del__(self):
        try:
            L.lib().rfl_schedule_destroy(self._h)
        except Exception:
            pass


class _CudaView:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}


def cuda_tensor(ptr: int, shape, np_dtype, device: int):
    """Zero-copy torch view over device memory owned by the loader."""
    import torch
    n = int(np.prod(shape))
    if n == 0 or not ptr:
        return torch.empty(shape, dtype=_torch_dtype(np_dtype), device=f"cuda:{device}")
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaView(ptr, shape, _TYPESTR[np_dtype]), device=f"cuda:{device}")
    return t


def _torch_dtype(np_dtype):
    import torch
    return {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32, np.uint8: torch.uint8,
            np.uint16: torch.int16, np.int64: torch.int64, np.uint64: torch.int64, np.uint32: torch.int32}[np_dtype]


@dataclass
class CsrBlock:
    """CsrBlock (block.hpp:58-64): u64 indptr (indptr[0]==0), u64 indices."""
    n_rows: int
    n_var: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray


@dataclass
class DenseBlock:
    """DenseBlock (block.hpp:23-27): row-major values."""
    n_rows: int
    n_var: int
    values: np.ndarray


@dataclass
class MiniBatch:
    """MiniBatch (loader.hpp:35-40)."""
    block: object
    global_indices: np.ndarray
    epoch_index: int = 0
    batch_index: int = 0


@dataclass
class DeviceBatch:
    """One minibatch on the GPU.  Tensors are views into the loader's ring."""
    epoch_index: int
    batch_index: int
    n_rows: int
    n_var: int
    layout: str
    global_indices: object      # torch int64 view of u64 ids
    global_indices_host: np.ndarray
    indptr: object = None       # torch int64 [n_rows+1] (csr)
    indices: object = None      # torch int32/int64 view of u32/u64 (csr)
    data: object = None         # csr values [nnz] or dense [n_rows, n_var]
    nnz: int = 0
    dtype: str = ""
    index_dtype: str = "u32"
    _ready_event: int = 0
    _d_gidx: int = 0

    def ids_to_host(self, dst: int, stream=None):
        """Queue the D2H copy of global_indices (u64[n_rows]) into host memory at
        address `dst` (pinned: asynchronous) on `stream` (a torch stream or a raw
        handle; default torch's current stream) -- rfl_ids_download_async."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        h = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        L.check(L.lib().rfl_ids_download_async(self._d_gidx, self.n_rows, dst, h))

    def to_minibatch(self) -> MiniBatch:
        """Host MiniBatch exactly as the reference returns it (u64 indices, raw value bytes)."""
        import torch
        torch.cuda.synchronize()
        g = self.global_indices_host.copy()
        if self.layout == "csr":
            ip = self.indptr.cpu().numpy().view(np.uint64)
            ix = self.indices.cpu().numpy()
            ix = ix.view(np.uint32 if self.index_dtype == "u32" else np.uint64).astype(np.uint64)
            dv = self.data.cpu().numpy()
            blk = CsrBlock(self.n_rows, self.n_var, ip, ix, dv)
        else:
            blk = DenseBlock(self.n_rows, self.n_var, self.data.cpu().numpy())
        return MiniBatch(blk, g, self.epoch_index, self.batch_index)


@dataclass
class LoaderCounters:
    """LoaderCounters (loader.hpp:42-45) + device staging counters."""
    blocks_fetched: int = 0
    read_ops: int = 0
    bytes_read: int = 0
    chunks_decoded: int = 0
    peak_buffer_rows: int = 0
    h2d_bytes: int = 0
    kernels_launched: int = 0
    decode_ms: float = 0.0    # time_kernels=True: device time of the staged-record expansion
    assembly_ms: float = 0.0  # ... and of the batch assembly kernels (finished batches)


class BatchIterator:
    """BatchIterator (loader.hpp:58-78) on a B200.

    output: "csr" (CSR store -> CSR batch, as the reference) or "dense"
    (CSR -> dense densify, or dense store rows); out_dtype "native"|"f32"|"bf16";
    transform None | "normalize_log1p" (library size to target_sum, then log1p).
    """

    def __init__(self, store, config: LoaderConfig, epoch_index: int = 0, *, device: int = 0,
                 staging: str = "resident", output: str | None = None, out_dtype: str = "native",
                 transform: str | None = None, target_sum: float = 1e4, out_slots: int = 2, stream=None,
                 time_kernels: bool = False, batches_per_launch: int = 1):
        if isinstance(store, DeviceStore):
            self.dstore = store
        else:
            self.dstore = DeviceStore(store if isinstance(store, StoreReader) else StoreReader(store), device,
                                      staging)
        man = self.dstore.manifest()
        self.device = self.dstore.device
        if output is None:
            output = "csr" if man.layout == "csr" else "dense"
        self.output = output
        self._epoch = epoch_index
        self.config = config
        dc = L.rfl_device_config(L.OUT_CSR if output == "csr" else L.OUT_DENSE, OUT_DTYPES[out_dtype],
                                 L.XF_NORMALIZE_LOG1P if transform == "normalize_log1p" else L.XF_NONE,
                                 float(target_sum), out_slots, L.DEV_TIME_KERNELS if time_kernels else 0,
                                 stream.cuda_stream if hasattr(stream, "cuda_stream") else (stream or None),
                                 int(batches_per_launch), 0)
        if transform not in (None, "normalize_log1p"):
            raise L.InvalidArgument(f"unknown transform {transform!r}")
        # stream=None: the loader assembles on its own stream, and every next() orders
        # torch's current stream after the batch (rfl_batch_wait), so `model(b.data)` or
        # `b.data.cpu()` never reads a buffer the kernel is still writing.  With an
        # explicit stream, batches are ordered on that stream only.
        self._own_stream = stream is None
        h = L.vp()
        L.check(L.lib().rfl_loader_create(self.dstore._h, C.byref(config._c()), epoch_index, C.byref(dc),
                                          C.byref(h)))
        self._h = h
        self._b = L.rfl_batch()
        self._many = (L.rfl_batch * 1)()
        self._views = {}
        self._hviews = {}

    def _view(self, ptr, shape, np_dtype, bf16=False):
        """cuda_tensor, cached: the loader's output slots are a fixed ring, so the
        same (pointer, shape) views come back every out_slots batches (bf16: the
        u16 view reinterpreted, cached as well)."""
        key = (ptr, shape, np_dtype, bf16)
        t = self._views.get(key)
        if t is None:
            if len(self._views) > 256:
                self._views.clear()
            t = cuda_tensor(ptr, shape, np_dtype, self.device)
            if bf16:
                import torch
                t = t.view(torch.bfloat16)
            self._views[key] = t
        return t

    def _host_view(self, addr, n):
        """numpy view of the loader's pinned host ids (a fixed ring like the device views)."""
        key = (addr, n)
        v = self._hviews.get(key)
        if v is None:
            if len(self._hviews) > 256:
                self._hviews.clear()
            v = self._hviews[key] = np.ctypeslib.as_array((C.c_uint64 * n).from_address(addr))
        return v

    def next(self) -> DeviceBatch | None:
        rc = L.check(L.lib().rfl_loader_next(self._h, C.byref(self._b)))
        if rc == L.END:
            return None
        return self._wrap(self._b)

    def next_many(self, k: int) -> list:
        """Up to k further batches in one call (fewer only at the end of the epoch;
        [] at the end).  With batches_per_launch = k they come from one launch."""
        if len(self._many) < k:
            self._many = (L.rfl_batch * k)()
        n = C.c_uint32()
        rc = L.check(L.lib().rfl_loader_next_many(self._h, self._many, k, C.byref(n)))
        if rc == L.END:
            return []
        return [self._wrap(self._many[i]) for i in range(n.value)]

    def _wrap(self, b) -> DeviceBatch:
        if self._own_stream:
            import torch
            L.check(L.lib().rfl_batch_wait(C.byref(b), C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        n = b.n_rows
        gh = self._host_view(b.h_gidx, n).copy() if n else np.zeros(0, np.uint64)
        g = self._view(b.d_gidx, (n,), np.int64)
        if b.layout == L.LAYOUT_CSR:
            idt = np.uint32 if b.index_dtype == L.IDX_U32 else np.uint64
            return DeviceBatch(b.epoch_index, b.batch_index, n, b.n_var, "csr", g, gh,
                               indptr=self._view(b.d_indptr, (n + 1,), np.int64),
                               indices=self._view(b.d_indices, (b.nnz,), np.int32 if idt == np.uint32 else np.int64),
                               data=self._view(b.d_data, (b.nnz,), _NP[b.dtype]), nnz=b.nnz,
                               dtype=str(b.dtype), index_dtype="u32" if idt == np.uint32 else "u64",
                               _ready_event=b.ready_event or 0, _d_gidx=b.d_gidx or 0)
        dt = b.dtype
        data = self._view(b.d_data, (n, b.n_var), _NP[dt], dt == L.BF16)
        return DeviceBatch(b.epoch_index, b.batch_index, n, b.n_var, "dense", g, gh, data=data, nnz=b.nnz,
                           dtype=str(dt), _ready_event=b.ready_event or 0, _d_gidx=b.d_gidx or 0)

    def __iter__(self):
        while (b := self.next()) is not None:
            yield b

    def counters(self) -> LoaderCounters:
        c = L.rfl_loader_counters()
        L.check(L.lib().rfl_loader_counters_get(self._h, C.byref(c)))
        return LoaderCounters(c.blocks_fetched, c.read_ops, c.bytes_read, c.chunks_decoded, c.peak_buffer_rows,
                              c.h2d_bytes, c.kernels_launched, c.decode_ms, c.assembly_ms)

    def peak_buffer_rows(self) -> int:
        return self.counters().peak_buffer_rows

    def epoch_index(self) -> int:
        return self._epoch

    def synchronize(self):
        L.check(L.lib().rfl_loader_sync(self._h))

    def close(self):
        if getattr(self, "_h", None):
            L.lib().rfl_loader_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def open_epoch(store, config: LoaderConfig, epoch_index: int, **device_kw) -> BatchIterator:
    """open_epoch (loader.cpp:312-315)."""
    return BatchIterator(store, config, epoch_index, **device_kw)
