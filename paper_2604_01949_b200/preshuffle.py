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


def run_shuffle(inputs, plan: ShufflePlan, out_path, out_config: ShuffleOutputConfig | None = None, *,
                device: int = 0, join: str = "outer", rank: int = 0, world: int = 1) -> ShuffleRunStats:
    """run_shuffle (preshuffle.cpp:185-378) with the round gather/permute/pack on the GPU.
    `inputs` is the ordered list of member store paths (DatasetCollection order)."""
    oc = out_config or ShuffleOutputConfig()
    if oc.codec != "none":
        raise L.InvalidArgument("GPU pre-shuffle writes codec none only")
    if inputs:
        from .store import StoreReader
        held = sum(StoreReader(p).manifest().n_obs for p in inputs)
        if plan.total_rows != held:  # preshuffle.cpp:191-194
            raise L.InvalidArgument(f"run_shuffle: plan covers {plan.total_rows} rows, collection holds {held}")
    paths = [str(p).encode() for p in inputs]
    arr = (C.c_char_p * len(paths))(*paths)
    cfg = L.rfl_shuffle_config(plan.block_rows, plan.buffer_rows, plan.seed, oc.chunk_rows, oc.chunks_per_shard,
                               -1 if oc.index_dtype is None else {"u32": 0, "u64": 1}[oc.index_dtype], device,
                               int(join == "outer"), rank, world, 0)
    st = L.rfl_shuffle_stats()
    L.check(L.lib().rfl_run_shuffle(arr, len(paths), str(out_path).encode(), C.byref(cfg), C.byref(st)))
    return ShuffleRunStats(st.peak_resident_rows, st.rows_written, st.rounds_executed, st.input_bytes_read,
                           st.h2d_bytes, st.d2h_bytes, st.gpu_ms)
