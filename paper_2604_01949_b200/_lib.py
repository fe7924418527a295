"""ctypes binding of the C-ABI in include/riffle_b200.h (libriffle_b200.so).

The shared library is built in-tree by ``paper_2604_01949_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libriffle_b200.so"

# status codes (riffle_b200.h)
OK, EINVAL, ECORRUPT, EIO, ECUDA, ENCCL, END, ENOMEM = range(8)
LAYOUT_DENSE, LAYOUT_CSR = 0, 1
F32, F64, I32, U8, BF16, NATIVE = 0, 1, 2, 3, 4, 255
IDX_U32, IDX_U64 = 0, 1
DEV_TIME_KERNELS = 1
STAGE_RESIDENT, STAGE_STREAM_PINNED, STAGE_STREAM_FILE, STAGE_RESIDENT_CODED = 0, 1, 2, 3
OUT_CSR, OUT_DENSE = 0, 1
XF_NONE, XF_NORMALIZE_LOG1P = 0, 1

u64 = C.c_uint64
u32 = C.c_uint32
vp = C.c_void_p
u64p = C.POINTER(C.c_uint64)


class rfl_store_info(C.Structure):
    _fields_ = [("format_version", u32), ("layout", u32), ("n_obs", u64), ("n_var", u64),
                ("value_dtype", u32), ("index_dtype", u32), ("chunk_rows", u64),
                ("chunks_per_shard", u64), ("codec", u32), ("has_provenance", u32)]


class rfl_synth_config(C.Structure):
    _fields_ = [("n_obs", u64), ("n_var", u64), ("layout", u32), ("value_dtype", u32),
                ("index_dtype", u32), ("codec", u32), ("density", C.c_double), ("seed", u64),
                ("chunk_rows", u64), ("chunks_per_shard", u64), ("threads", u32), ("one_hot", u32),
                ("counts", u32), ("reserved", u32)]


class rfl_loader_config(C.Structure):
    _fields_ = [("fetch_block_rows", u64), ("buffer_capacity_rows", u64), ("batch_rows", u64),
                ("seed", u64), ("prefetch_depth", u32), ("drop_last", u32), ("cache_bypass", u32),
                ("rank", u32), ("world", u32), ("even_batches", u32)]


class rfl_device_config(C.Structure):
    _fields_ = [("output", u32), ("out_dtype", u32), ("transform", u32), ("target_sum", C.c_float),
                ("out_slots", u32), ("flags", u32), ("stream", vp), ("batches_per_launch", u32),
                ("reserved2", u32)]


class rfl_batch(C.Structure):
    _fields_ = [("epoch_index", u64), ("batch_index", u64), ("n_rows", u64), ("nnz", u64), ("n_var", u64),
                ("layout", u32), ("dtype", u32), ("index_dtype", u32), ("reserved", u32),
                ("d_gidx", vp), ("d_indptr", vp), ("d_indices", vp), ("d_data", vp),
                ("h_gidx", vp), ("ready_event", vp)]  # h_gidx: const uint64_t* (read as an address)


class rfl_loader_counters(C.Structure):
    _fields_ = [("blocks_fetched", u64), ("read_ops", u64), ("bytes_read", u64), ("chunks_decoded", u64),
                ("peak_buffer_rows", u64), ("h2d_bytes", u64), ("kernels_launched", u64),
                ("decode_ms", C.c_double), ("assembly_ms", C.c_double)]


class rfl_rowref(C.Structure):
    _fields_ = [("rec_off", u64), ("gidx", u64)]


class rfl_arena_desc(C.Structure):
    _fields_ = [("base", vp), ("chunk_rows", u64), ("n_var", u64), ("layout", u32), ("value_dtype", u32),
                ("index_dtype", u32), ("reserved", u32)]


class rfl_shuffle_config(C.Structure):
    _fields_ = [("block_rows", u64), ("buffer_rows", u64), ("seed", u64), ("out_chunk_rows", u64),
                ("out_chunks_per_shard", u64), ("out_index_dtype", C.c_int32), ("device", C.c_int32),
                ("join_outer", u32), ("rank", u32), ("world", u32), ("reserved", u32)]


class rfl_shuffle_stats(C.Structure):
    _fields_ = [("peak_resident_rows", u64), ("rows_written", u64), ("rounds_executed", u64),
                ("input_bytes_read", u64), ("h2d_bytes", u64), ("d2h_bytes", u64), ("gpu_ms", C.c_double),
                ("send_ms", C.c_double), ("peer_bytes", u64)]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = [
    ("rfl_last_error", C.c_char_p, []),
    ("rfl_version", C.c_char_p, []),
    ("rfl_device_count", C.c_int, []),
    ("rfl_store_open", C.c_int, [C.c_char_p, C.POINTER(vp)]),
    ("rfl_store_get_info", C.c_int, [vp, C.POINTER(rfl_store_info)]),
    ("rfl_store_record_size", C.c_int, [vp, u64, u64p]),
    ("rfl_store_read_record", C.c_int, [vp, u64, vp, u64]),
    ("rfl_store_close", None, [vp]),
    ("rfl_synth_store", C.c_int, [C.c_char_p, C.POINTER(rfl_synth_config)]),
    ("rfl_loader_config_validate", C.c_int, [C.POINTER(rfl_loader_config)]),
    ("rfl_plan_epoch", C.c_int, [u64, C.POINTER(rfl_loader_config), u64, vp, vp]),
    ("rfl_schedule_create", C.c_int, [u64, C.POINTER(rfl_loader_config), u64, C.POINTER(vp)]),
    ("rfl_schedule_next", C.c_int, [vp, vp, u64p]),
    ("rfl_schedule_stats", C.c_int, [vp, u64p, u64p]),
    ("rfl_schedule_destroy", None, [vp]),
    ("rfl_dstore_create", C.c_int, [vp, C.c_int, u32, C.POINTER(vp)]),
    ("rfl_dstore_arena", C.c_int, [vp, C.POINTER(vp), C.POINTER(u64p), u64p]),
    ("rfl_dstore_destroy", None, [vp]),
    ("rfl_loader_create", C.c_int, [vp, C.POINTER(rfl_loader_config), u64, C.POINTER(rfl_device_config),
                                    C.POINTER(vp)]),
    ("rfl_loader_next", C.c_int, [vp, C.POINTER(rfl_batch)]),
    ("rfl_loader_counters_get", C.c_int, [vp, C.POINTER(rfl_loader_counters)]),
    ("rfl_batch_download", C.c_int, [C.POINTER(rfl_batch), vp, vp, vp, vp]),
    ("rfl_batch_wait", C.c_int, [C.POINTER(rfl_batch), vp]),
    ("rfl_ids_download_async", C.c_int, [vp, u64, vp, vp]),
    ("rfl_loader_next_many", C.c_int, [vp, C.POINTER(rfl_batch), u32, C.POINTER(u32)]),
    ("rfl_device_can_access_peer", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_int)]),
    ("rfl_loader_sync", C.c_int, [vp]),
    ("rfl_dstore_bytes", C.c_int, [vp, u64p, u64p]),
    ("rfl_loader_destroy", None, [vp]),
    ("rfl_csr_gather", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, vp, vp, vp, vp, vp]),
    ("rfl_csr_gather_prefixed", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, vp, vp, vp, vp, vp]),
    ("rfl_csr_densify", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, u32, u32, C.c_float, vp, vp, vp]),
    ("rfl_dense_gather", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, u32, vp, vp, vp]),
    ("rfl_onehot_gather", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, u32, vp, vp, vp]),
    ("rfl_csr_scan", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, vp, vp]),
    ("rfl_csr_pack", C.c_int, [C.POINTER(rfl_arena_desc), vp, u64, u64, u32, vp, vp, vp]),
    ("rfl_plan_shuffle", C.c_int, [u64, u64, u64, u64, u64p, vp, vp]),
    ("rfl_shuffle_order", C.c_int, [u64, u64, u64, u64, vp]),
    ("rfl_shuffle_round_routes", C.c_int, [u64, u64, u64, u64, u64, u64, u32, u64, u64p, u64p, vp, vp, vp]),
    ("rfl_pshuf_create", C.c_int, [C.POINTER(C.c_char_p), u64, C.c_char_p, C.POINTER(rfl_shuffle_config),
                                   C.POINTER(vp), u64p]),
    ("rfl_pshuf_stage", C.c_int, [vp, u64, vp]),
    ("rfl_pshuf_recv_buffer", C.c_int, [vp, u64, C.POINTER(vp), vp, C.POINTER(C.c_int)]),
    ("rfl_pshuf_send", C.c_int, [vp, u64, C.POINTER(vp)]),
    ("rfl_pshuf_emit", C.c_int, [vp, u64, vp]),
    ("rfl_pshuf_finish", C.c_int, [vp, C.POINTER(rfl_shuffle_stats)]),
    ("rfl_pshuf_destroy", None, [vp]),
    ("rfl_ipc_open", C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    ("rfl_ipc_close", C.c_int, [vp, C.c_int]),
    ("rfl_run_shuffle", C.c_int, [C.POINTER(C.c_char_p), u64, C.c_char_p, C.POINTER(rfl_shuffle_config),
                                  C.POINTER(rfl_shuffle_stats)]),
]

_lib = None


def lib():
    """Load libriffle_b200.so (no fallback: raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing — run __graft_entry__.build() "
                              "(make -C paper_2604_01949_b200/csrc); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


# ----------------------------------------------------------------- errors ---
class RiffleError(RuntimeError):
    """riffle::Error (error.hpp:9-12)."""


class InvalidArgument(RiffleError, ValueError):
    """riffle::InvalidArgument (error.hpp:16-19)."""


class CorruptStore(RiffleError):
    """riffle::CorruptStore (error.hpp:23-26)."""


class IoError(RiffleError, OSError):
    """riffle::IoError (error.hpp:29-32)."""


class CudaError(RiffleError):
    """Device failure (new; the reference has no device)."""


class NcclError(RiffleError):
    """Collective failure on the pre-shuffle's exchange (new)."""


class OutOfMemory(RiffleError, MemoryError):
    """Host (std::bad_alloc) or device (cudaErrorMemoryAllocation) allocation failure (new)."""


_EXC = {EINVAL: InvalidArgument, ECORRUPT: CorruptStore, EIO: IoError, ECUDA: CudaError, ENCCL: NcclError,
        ENOMEM: OutOfMemory}


def check(rc: int) -> int:
    if rc in (OK, END):
        return rc
    msg = lib().rfl_last_error().decode(errors="replace")
    raise _EXC.get(rc, RiffleError)(msg)
