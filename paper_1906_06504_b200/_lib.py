"""ctypes binding of the C ABI in include/batchheap_b200.h.

The library ``libbatchheap_b200.so`` is built in-tree by
``__graft_entry__.build()`` (``make -C paper_1906_06504_b200/csrc``).  There
is no fallback: if the library is missing this module raises on import of any
entry point, and ``bh_create`` refuses to run without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BH_LIB") or os.path.join(HERE, "libbatchheap_b200.so")

BH_OK, BH_E_CONFIG, BH_E_CAPACITY, BH_E_EMPTY, BH_E_INVALID_KEY, BH_E_CUDA, BH_E_INTERNAL = range(7)
BH_TD, BH_BU = 0, 1
BH_FLAG_ELIDE_MERGES = 0x1
BH_FLAG_RECORD = 0x2
BH_FLAG_PROFILE = 0x4
BH_OP_INSERT, BH_OP_DELETE = 0, 1
BH_RUN_EXPLICIT_STREAM = 0x1


class bh_peek(C.Structure):
    _fields_ = [("node_count", C.c_uint64), ("key_count", C.c_uint64),
                ("partial_len", C.c_uint64), ("level_count", C.c_uint64)]


COUNTER_FIELDS = ("inserts", "deletes", "merges", "elided_merges", "early_stops",
                  "propagation_node_visits", "coop_handoffs", "max_partial_len")


class bh_counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in COUNTER_FIELDS]


class bh_op(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("len", C.c_uint32), ("offset", C.c_uint64)]


class bh_run_cfg(C.Structure):
    _fields_ = [("ctas", C.c_uint32), ("flags", C.c_uint32), ("stream", C.c_void_p)]


class bh_sssp_cfg(C.Structure):
    _fields_ = [("threshold", C.c_uint64), ("heap_node_capacity", C.c_uint32), ("ctas", C.c_uint32),
                ("reserved", C.c_uint64)]


class bh_sssp_stats(C.Structure):
    _fields_ = [("visits", C.c_uint64), ("rounds", C.c_uint64), ("keys_through_heap", C.c_uint64),
                ("seconds", C.c_double)]


class bh_bb_cfg(C.Structure):
    _fields_ = [("gc_threshold", C.c_uint64), ("heap_node_capacity", C.c_uint32), ("ctas", C.c_uint32),
                ("pop_ops", C.c_uint32), ("reserved", C.c_uint32), ("arena_nodes", C.c_uint64),
                ("max_explored", C.c_uint64)]


class bh_bb_outcome(C.Structure):
    _fields_ = [("best", C.c_uint64), ("explored", C.c_uint64), ("gc_passes", C.c_uint64),
                ("rounds", C.c_uint64), ("arena_nodes", C.c_uint64), ("seconds", C.c_double)]


class bh_event(C.Structure):
    _fields_ = [("ts", C.c_uint64), ("op", C.c_uint32), ("kind", C.c_uint16),
                ("pad", C.c_uint16), ("node", C.c_uint64)]


# Every symbol include/batchheap_b200.h declares: name -> (restype, argtypes)
_vp, _u32, _u64, _i = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
SIGNATURES = {
    "bh_create": (_i, [C.POINTER(_vp), _i, _u32, _u32, _u32, _u32, _i]),
    "bh_destroy": (None, [_vp]),
    "bh_insert": (_i, [_vp, _vp, _u32]),
    "bh_delete_min": (_i, [_vp, _vp, C.POINTER(_u32)]),
    "bh_run_ops": (_i, [_vp, _vp, _u64, _vp, _u64, _vp, _u64, _vp, _vp, _vp, C.POINTER(bh_run_cfg)]),
    "bh_run_ops_device": (_i, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, C.POINTER(bh_run_cfg)]),
    "bh_plan_phase": (_i, [_vp, _i, _u64, _vp, _i, _vp]),
    "bh_peek_stats": (_i, [_vp, C.POINTER(bh_peek)]),
    "bh_get_counters": (_i, [_vp, C.POINTER(bh_counters)]),
    "bh_reset_counters": (_i, [_vp]),
    "bh_select_insert_target": (_i, [_vp, C.POINTER(_u64)]),
    "bh_collect_resident": (_i, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "bh_check_invariants": (_i, [_vp, C.POINTER(_i), C.c_char_p, C.c_size_t]),
    "bh_dump": (_i, [_vp, _vp, _u64, _vp, C.POINTER(_u32), _vp]),
    "bh_info": (_i, [_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_u32),
                     C.POINTER(_i), C.POINTER(_u32), C.POINTER(_u32)]),
    "bh_history": (_i, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "bh_profile": (_i, [_vp, C.POINTER(_u64), _u32, _i]),
    "bh_last_error": (C.c_char_p, []),
    "bh_sort_batches": (_i, [_u32, _u32, _vp, _vp, _u64, _vp]),
    "bh_merge_split": (_i, [_u32, _u32, _vp, _vp, _vp, _vp, _u64, _vp]),
    "bh_slot_for_rank": (_u64, [_u64]),
    "bh_bit_reverse": (_u64, [_u64, C.c_uint]),
    "bh_generate_keys": (_i, [_i, _u64, _u64, _u32, _vp]),
    "bh_build_info": (C.c_char_p, []),
    "bh_plan_batches": (_i, [_u32, _u64, _u32, _u32, _u64, _vp, _vp, _u64, C.POINTER(_u64)]),
    "bh_grid_graph_edges": (_u64, [_u32, _u32]),
    "bh_grid_graph": (_i, [_u32, _u32, _u64, _vp, _vp, _vp]),
    "bh_sssp": (_i, [_u32, _vp, _vp, _vp, _u32, C.POINTER(bh_sssp_cfg), _i, _vp, C.POINTER(bh_sssp_stats)]),
    "bh_generate_knapsack": (_u64, [_i, _u32, _u32, _u64, _vp, _vp]),
    "bh_knapsack_bb": (_i, [_u32, _vp, _vp, _u64, C.POINTER(bh_bb_cfg), _i, C.POINTER(bh_bb_outcome)]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load the C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                        "(make -C paper_1906_06504_b200/csrc); there is no CPU fallback")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def last_error() -> str:
    msg = lib().bh_last_error()
    return msg.decode() if msg else ""
