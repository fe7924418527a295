"""riffle on B200: GPU-native chunked minibatch assembly and pre-shuffle for
riffle stores (the C++ restatement of annbatch, arXiv 2604.01949).

The public surface mirrors the reference C++ API (proj/core/include/riffle):
LoaderConfig / plan_epoch / BatchIterator / open_epoch / MiniBatch,
plan_shuffle / run_shuffle, StoreReader / synth_store.  Every call goes through
the C-ABI of libriffle_b200.so (include/riffle_b200.h); there is no CPU
fallback.
"""
from ._lib import (CorruptStore, CudaError, InvalidArgument, IoError, NcclError, OutOfMemory,  # noqa: F401
                   RiffleError, lib)
from .loader import (BatchIterator, CsrBlock, DenseBlock, DeviceBatch, EpochPlan, EpochSchedule,  # noqa: F401
                     LoaderConfig, LoaderCounters, MiniBatch, open_epoch, plan_epoch)
from .preshuffle import (ShuffleOutputConfig, ShufflePlan, ShuffleRunStats, plan_shuffle, run_shuffle,  # noqa: F401
                         shuffle_order)
from .store import DeviceStore, StoreManifest, StoreReader, SynthConfig, synth_store  # noqa: F401

__version__ = "0.1.0"
