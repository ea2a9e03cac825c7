"""B200-native batched generalized heap (arXiv 1906.06504).

Host mirror of the reference's ``batchheap::GeneralizedHeap`` over the C ABI
in ``include/batchheap_b200.h``; the heap itself runs as hand-written sm_100a
kernels in ``libbatchheap_b200.so``.
"""
from .heap import (  # noqa: F401
    CapacityError,
    ConfigError,
    DeviceError,
    EmptyHeapError,
    GeneralizedHeap,
    HeapCounters,
    HeapOptions,
    HeapPeek,
    InvariantReport,
    OP_DTYPE,
    RunResult,
    Variant,
    bit_reverse,
    generate_keys,
    make_ops,
    merge_split_device,
    path_to_slot,
    phase_ops,
    slot_for_rank,
    sort_batches_device,
)
from ._lib import LIB_PATH, SIGNATURES  # noqa: F401
