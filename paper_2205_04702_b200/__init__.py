"""B200-native ScratchPipe (arXiv 2205.04702): a look-forward embedding
scratchpad for recommendation-model training.

The hot path lives in ``lib/libscratchpipe.so`` (hand-written sm_100a CUDA
kernels + a C++ runtime behind the C ABI in ``include/scratchpipe.h``);
this package is the thin Python binding over it plus host-side helpers
(sizing, table-wise sharding for multi-GPU).  No CPU fallback exists.
"""
from ._binding import (  # noqa: F401
    KERNEL_KINDS,
    LIB_PATH,
    SP_ERR_CAPACITY,
    SP_ERR_INDEX_RANGE,
    SP_ERR_INVALID_ARG,
    SP_ERR_STATE,
    SP_OK,
    STATUS_NAMES,
    HostTable,
    ScratchPipe,
    SpError,
    header_symbols,
    lib,
    nccl_unique_id,
    shard_plan,
)
from .sizing import slots_for_fraction, window_batches, worst_case_storage_bytes  # noqa: F401

__all__ = ["ScratchPipe", "SpError", "lib", "header_symbols", "worst_case_storage_bytes",
           "slots_for_fraction", "window_batches"]
