"""Store handles — host mirror of riffle's StoreReader / synth_store
(reference include/riffle/store.hpp:136-170, include/riffle/synth.hpp:15-39)
plus the device-side store image (new)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib as L

LAYOUTS = {"dense": L.LAYOUT_DENSE, "csr": L.LAYOUT_CSR}
VDTYPES = {"f32": L.F32, "f64": L.F64, "i32": L.I32, "u8": L.U8}
IDTYPES = {"u32": L.IDX_U32, "u64": L.IDX_U64}
STAGING = {"resident": L.STAGE_RESIDENT, "stream_pinned": L.STAGE_STREAM_PINNED,
           "stream_file": L.STAGE_STREAM_FILE, "resident_coded": L.STAGE_RESIDENT_CODED}
_INV = lambda d: {v: k for k, v in d.items()}  # noqa: E731


@dataclass
class StoreManifest:
    """StoreManifest (manifest.hpp:16-54), without var_names."""
    format_version: int
    layout: str
    n_obs: int
    n_var: int
    value_dtype: str
    index_dtype: str | None
    chunk_rows: int
    chunks_per_shard: int
    codec: str
    has_provenance: bool

    def chunk_count(self) -> int:
        return (self.n_obs + self.chunk_rows - 1) // self.chunk_rows

    def rows_in_chunk(self, chunk: int) -> int:
        s = chunk * self.chunk_rows
        return min(self.chunk_rows, self.n_obs - s)


class StoreReader:
    """Read handle over a finished store (store.hpp:136-170).  Opening validates
    the manifest; shard footers are validated lazily, as in the reference."""

    def __init__(self, root):
        self.root = str(root)
        h = L.vp()
        L.check(L.lib().rfl_store_open(self.root.encode(), C.byref(h)))
        self._h = h
        info = L.rfl_store_info()
        L.check(L.lib().rfl_store_get_info(self._h, C.byref(info)))
        lay = _INV(LAYOUTS)[info.layout]
        self._manifest = StoreManifest(info.format_version, lay, info.n_obs, info.n_var,
                                       _INV(VDTYPES)[info.value_dtype],
                                       _INV(IDTYPES)[info.index_dtype] if lay == "csr" else None,
                                       info.chunk_rows, info.chunks_per_shard,
                                       "none" if info.codec == 0 else "deflate", bool(info.has_provenance))

    def manifest(self) -> StoreManifest:
        return self._manifest

    def read_record(self, chunk: int) -> bytes:
        """Raw (undecoded) chunk record bytes (SURVEY §8b "missing lower-level API")."""
        n = C.c_uint64()
        L.check(L.lib().rfl_store_record_size(self._h, chunk, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        L.check(L.lib().rfl_store_read_record(self._h, chunk, buf, n.value))
        return buf.raw

    def close(self):
        if getattr(self, "_h", None):
            L.lib().rfl_store_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SynthConfig:
    """SynthConfig (synth.hpp:15-27)."""
    n_obs: int = 0
    n_var: int = 0
    layout: str = "dense"
    value_dtype: str = "f32"
    index_dtype: str = "u32"
    density: float = 0.01
    seed: int = 0
    chunk_rows: int = 1024
    chunks_per_shard: int = 128
    codec: str = "none"
    threads: int = 0
    one_hot: int = 0  # > 0: procedural one-hot dense u8 rows (channel planes), see rfl_synth_config
    counts: bool = False  # procedural counts-like csr rows (2k-4k nnz/row, values 1..64), see rfl_synth_config


def synth_store(path, config: SynthConfig) -> StoreManifest:
    """synth_store (synth.cpp:60-144): byte-identical to the reference for equal configs."""
    c = L.rfl_synth_config(config.n_obs, config.n_var, LAYOUTS[config.layout], VDTYPES[config.value_dtype],
                           IDTYPES[config.index_dtype], 0 if config.codec == "none" else 1, config.density,
                           config.seed, config.chunk_rows, config.chunks_per_shard, config.threads,
                           config.one_hot, int(config.counts), 0)
    L.check(L.lib().rfl_synth_store(str(path).encode(), C.byref(c)))
    return StoreReader(path).manifest()


class DeviceStore:
    """A store image on one GPU, shared by many iterators (loader.hpp:55-57).

    staging: "resident" (all chunk records in HBM), "stream_pinned" (records in
    pinned host memory, blocks cudaMemcpyAsync'd per fetch) or "stream_file"
    (pread into pinned staging per fetch)."""

    def __init__(self, reader: StoreReader | str, device: int = 0, staging: str = "resident"):
        self.reader = reader if isinstance(reader, StoreReader) else StoreReader(reader)
        self.device = device
        self.staging = staging
        h = L.vp()
        L.check(L.lib().rfl_dstore_create(self.reader._h, device, STAGING[staging], C.byref(h)))
        self._h = h

    def manifest(self) -> StoreManifest:
        return self.reader.manifest()

    def image_bytes(self):
        """(decoded record bytes of the store, bytes of its re-encoded staging image or 0)."""
        r, s = C.c_uint64(), C.c_uint64()
        L.check(L.lib().rfl_dstore_bytes(self._h, C.byref(r), C.byref(s)))
        return r.value, s.value

    def arena(self):
        """(device base pointer, per-chunk record offsets) of a resident image."""
        base, offs, n = L.vp(), L.u64p(), C.c_uint64()
        L.check(L.lib().rfl_dstore_arena(self._h, C.byref(base), C.byref(offs), C.byref(n)))
        import numpy as np
        return base.value, np.ctypeslib.as_array(offs, shape=(n.value,)).copy()

    def arena_desc(self) -> L.rfl_arena_desc:
        m = self.manifest()
        base, _ = self.arena()
        return L.rfl_arena_desc(base, m.chunk_rows, m.n_var, LAYOUTS[m.layout], VDTYPES[m.value_dtype],
                                IDTYPES[m.index_dtype] if m.index_dtype else 0, 0)

    def close(self):
        if getattr(self, "_h", None):
            L.lib().rfl_dstore_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
