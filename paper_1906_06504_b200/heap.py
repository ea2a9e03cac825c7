"""Host mirror of the reference's heap API over the C ABI.

``GeneralizedHeap`` keeps the shape of ``batchheap::GeneralizedHeap``
(reference proj/include/batchheap/heap.hpp:72-181): the same constructor
arguments, methods, return values and exception types, so the parity tests
read like the reference's own tests (proj/tests/test_heap.cpp).  Every call
goes through ``libbatchheap_b200.so`` to the sm_100a kernels; nothing here
computes heap results on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


# ------------------------------------------------------------- errors ----
class ConfigError(RuntimeError):
    """batchheap::ConfigError (proj/include/batchheap/batch.hpp:23-25)."""


class CapacityError(RuntimeError):
    """batchheap::CapacityError (proj/include/batchheap/batch.hpp:26-28)."""


class EmptyHeapError(RuntimeError):
    """batchheap::EmptyHeapError (proj/include/batchheap/batch.hpp:29-31)."""


class DeviceError(RuntimeError):
    """CUDA/runtime failure (no reference analogue)."""


def _raise(code: int):
    if code == L.BH_OK:
        return
    msg = L.last_error()
    if code == L.BH_E_CONFIG:
        raise ConfigError(msg)
    if code == L.BH_E_CAPACITY:
        raise CapacityError(msg)
    if code == L.BH_E_EMPTY:
        raise EmptyHeapError(msg)
    if code == L.BH_E_INVALID_KEY:
        raise ValueError(msg)  # std::invalid_argument (proj/src/batch.cpp:13-15)
    if code == L.BH_E_CUDA:
        raise DeviceError(msg)
    raise RuntimeError(msg)  # std::logic_error (proj/src/heap.cpp:462-463)


class Variant(enum.IntEnum):
    """batchheap::Variant (proj/include/batchheap/history.hpp:23)."""
    TD = L.BH_TD
    BU = L.BH_BU


@dataclass
class HeapOptions:
    """batchheap::HeapOptions (proj/include/batchheap/heap.hpp:43-47)."""
    elide_merges: bool = True


@dataclass
class HeapCounters:
    inserts: int = 0
    deletes: int = 0
    merges: int = 0
    elided_merges: int = 0
    early_stops: int = 0
    propagation_node_visits: int = 0
    coop_handoffs: int = 0
    max_partial_len: int = 0


@dataclass
class HeapPeek:
    node_count: int = 0
    key_count: int = 0
    partial_len: int = 0
    level_count: int = 0


@dataclass
class InvariantReport:
    ok: bool = True
    detail: str = ""


@dataclass
class RunResult:
    """Outputs of one bulk submission (numpy, host)."""
    out: np.ndarray
    status: np.ndarray
    lens: np.ndarray
    seq: np.ndarray


def _key_dtype(bits: int):
    return np.uint32 if bits == 32 else np.uint64


class GeneralizedHeap:
    """B200 generalized heap; mirrors batchheap::GeneralizedHeap.

    ``key_bits`` (32 or 64) selects the device key width; the reference's Key
    is 64-bit (proj/include/batchheap/batch.hpp:17).  ``record=True`` enables
    the device event log used by the linearizability checkers (the
    reference's ``Recorder*`` argument)."""

    def __init__(self, variant: Variant, k: int, max_nodes: int,
                 options: Optional[HeapOptions] = None, record: bool = False,
                 key_bits: int = 64, device: int = 0, profile: bool = False,
                 debug_flags: int = 0):
        options = options or HeapOptions()
        flags = (L.BH_FLAG_ELIDE_MERGES if options.elide_merges else 0) | \
                (L.BH_FLAG_RECORD if record else 0) | (L.BH_FLAG_PROFILE if profile else 0) | \
                int(debug_flags)
        h = C.c_void_p()
        _raise(L.lib().bh_create(C.byref(h), int(variant), int(k), int(max_nodes),
                                 int(key_bits), flags, int(device)))
        self._h = h
        self._variant = Variant(variant)
        self._k = int(k)
        self._max_nodes = int(max_nodes)
        self.key_bits = int(key_bits)
        self.dtype = _key_dtype(key_bits)
        self.options = options
        self.recording = record
        info = self.info()
        self.slot_count = info["slot_count"]
        self.threads_per_cta = info["threads_per_cta"]
        self.max_ctas = info["max_ctas"]

    def close(self):
        if getattr(self, "_h", None):
            L.lib().bh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -------------------------------------------------------------- ops --
    def insert(self, items: Sequence[int]) -> None:
        """insert (heap.hpp:81-83): 1..k keys, all below the sentinel."""
        a = np.ascontiguousarray(np.asarray(items, dtype=np.uint64))
        if self.key_bits == 32:
            if a.size and int(a.max()) > 0xFFFFFFFF:
                raise ValueError("key does not fit the 32-bit heap")
            a = a.astype(np.uint32)
        _raise(L.lib().bh_insert(self._h, a.ctypes.data_as(C.c_void_p), a.size))

    def try_delete_min(self) -> Optional[np.ndarray]:
        """try_delete_min (heap.hpp:88): None on an empty heap."""
        out = np.empty(self._k, dtype=self.dtype)
        n = C.c_uint32(0)
        code = L.lib().bh_delete_min(self._h, out.ctypes.data_as(C.c_void_p), C.byref(n))
        if code == L.BH_E_EMPTY:
            return None
        _raise(code)
        return out[:n.value].astype(np.uint64)

    def delete_min(self) -> np.ndarray:
        """delete_min (heap.hpp:86): raises EmptyHeapError when empty."""
        r = self.try_delete_min()
        if r is None:
            raise EmptyHeapError("delete_min: heap empty")
        return r

    # ------------------------------------------------------------ bulk --
    def run_ops(self, ops: np.ndarray, key_pool: np.ndarray, out_len: int, ctas: int = 0) -> RunResult:
        """Bulk submission through bh_run_ops with HOST buffers.

        ``ops`` is a structured array with fields kind/len/offset (see
        ``make_ops``)."""
        ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
        pool = np.ascontiguousarray(key_pool, dtype=self.dtype)
        out = np.empty(max(out_len, 1), dtype=self.dtype)
        status = np.empty(len(ops), dtype=np.uint32)
        lens = np.empty(len(ops), dtype=np.uint32)
        seq = np.empty(len(ops), dtype=np.uint64)
        cfg = L.bh_run_cfg(ctas, 0, None)
        _raise(L.lib().bh_run_ops(self._h, ops.ctypes.data_as(C.c_void_p), len(ops),
                                  pool.ctypes.data_as(C.c_void_p), pool.size,
                                  out.ctypes.data_as(C.c_void_p), out_len,
                                  status.ctypes.data_as(C.c_void_p), lens.ctypes.data_as(C.c_void_p),
                                  seq.ctypes.data_as(C.c_void_p), C.byref(cfg)))
        return RunResult(out[:out_len], status, lens, seq)

    def run_ops_ptr(self, ops_ptr: int, n_ops: int, pool_ptr: int, out_ptr: int,
                    status_ptr: int = 0, lens_ptr: int = 0, seq_ptr: int = 0,
                    ctas: int = 0, stream: Optional[int] = None) -> None:
        """Bulk submission with DEVICE pointers (e.g. torch ``data_ptr()``),
        asynchronous on ``stream`` (a cudaStream_t as int; 0 is the legacy
        default stream; None the handle's own stream)."""
        cfg = L.bh_run_cfg(ctas, 0 if stream is None else L.BH_RUN_EXPLICIT_STREAM, stream or None)
        _raise(L.lib().bh_run_ops_device(self._h, ops_ptr, n_ops, pool_ptr or None, out_ptr or None,
                                         status_ptr or None, lens_ptr or None, seq_ptr or None,
                                         C.byref(cfg)))

    def run_ops_host_ptr(self, ops_ptr: int, n_ops: int, pool_ptr: int, pool_len: int,
                         out_ptr: int, out_len: int, status_ptr: int = 0, lens_ptr: int = 0,
                         seq_ptr: int = 0, ctas: int = 0, stream: int = 0) -> None:
        """Bulk submission with HOST pointers (pinned buffers), synchronous."""
        cfg = L.bh_run_cfg(ctas, 0, stream or None)
        _raise(L.lib().bh_run_ops(self._h, ops_ptr, n_ops, pool_ptr or None, pool_len,
                                  out_ptr or None, out_len, status_ptr or None, lens_ptr or None,
                                  seq_ptr or None, C.byref(cfg)))

    def plan_phase_ptr(self, kind: int, n_keys: int, ops_ptr: int, on_device: bool, stream: int = 0):
        _raise(L.lib().bh_plan_phase(self._h, kind, n_keys, ops_ptr, int(on_device), stream or None))

    # ---------------------------------------------------- introspection --
    def peek_stats(self) -> HeapPeek:
        p = L.bh_peek()
        _raise(L.lib().bh_peek_stats(self._h, C.byref(p)))
        return HeapPeek(p.node_count, p.key_count, p.partial_len, p.level_count)

    def counters(self) -> HeapCounters:
        c = L.bh_counters()
        _raise(L.lib().bh_get_counters(self._h, C.byref(c)))
        return HeapCounters(*(getattr(c, n) for n in L.COUNTER_FIELDS))

    def reset_counters(self) -> None:
        _raise(L.lib().bh_reset_counters(self._h))

    def select_insert_target(self) -> int:
        s = C.c_uint64(0)
        _raise(L.lib().bh_select_insert_target(self._h, C.byref(s)))
        return s.value

    def collect_resident(self) -> np.ndarray:
        n = C.c_uint64(0)
        _raise(L.lib().bh_collect_resident(self._h, None, 0, C.byref(n)))
        out = np.empty(max(n.value, 1), dtype=self.dtype)
        _raise(L.lib().bh_collect_resident(self._h, out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
        return out[:n.value].astype(np.uint64)

    def check_invariants(self) -> InvariantReport:
        ok = C.c_int(0)
        buf = C.create_string_buffer(4096)
        _raise(L.lib().bh_check_invariants(self._h, C.byref(ok), buf, 4096))
        return InvariantReport(bool(ok.value), buf.value.decode())

    def dump(self):
        """Raw device layout: (keys[slot_count, k] in slot order, partial, states[slot_count+1])."""
        keys = np.empty(self.slot_count * self._k, dtype=self.dtype)
        part = np.empty(self._k, dtype=self.dtype)
        plen = C.c_uint32(0)
        states = np.empty(self.slot_count + 1, dtype=np.uint32)
        _raise(L.lib().bh_dump(self._h, keys.ctypes.data_as(C.c_void_p), keys.size,
                               part.ctypes.data_as(C.c_void_p), C.byref(plen),
                               states.ctypes.data_as(C.c_void_p)))
        return keys.reshape(self.slot_count, self._k), part[:plen.value].copy(), states

    def history_events(self) -> np.ndarray:
        """Device event log of the last bulk run (RECORD heaps)."""
        n = C.c_uint64(0)
        _raise(L.lib().bh_history(self._h, None, 0, C.byref(n)))
        ev = np.empty(max(n.value, 1), dtype=EVENT_DTYPE)
        _raise(L.lib().bh_history(self._h, ev.ctypes.data_as(C.c_void_p), ev.size, C.byref(n)))
        return ev[:n.value]

    PROFILE_FIELDS = ("ins_ops", "ins_sort", "ins_root_wait", "ins_root_hold", "ins_rest",
                      "del_ops", "del_root_wait", "del_root_hold", "del_rest", "child_wait",
                      "levels", "cta_cycles", "rs_head", "rs_child", "rs_last", "rs_load",
                      "rs_fill", "lv_acq", "lv_load", "lv_merge", "lv_rel", "served",
                      "serve_holds", "bu_parent", "bu_retake", "bu_levels", "split_a", "split_b",
                      "del_served", "del_serve_holds", "sv_split", "sv_a", "sv_b", "sv_r1", "sv_r2",
                      "sv_r3", "sv_next", "sv_claim", "s3_ops", "s3_op", "s3_r0", "s3_wait_rf",
                      "s3_r1", "s3_wait_c3", "s3_r2", "s3_r3", "s3_claim", "s3_refill", "s3_ctl",
                      "s3_rec", "s3_wake", "s3_post", "s3_start", "hold_cs", "hold_cs_n", "climb_root",
                      "climb_root_n", "cs1", "cs2", "cs3", "cs4")

    def profile(self, reset: bool = True) -> dict:
        """SM-cycle profile of a BH_FLAG_PROFILE heap (see bh_profile)."""
        buf = (C.c_uint64 * 64)()
        _raise(L.lib().bh_profile(self._h, buf, 64, int(reset)))
        return dict(zip(self.PROFILE_FIELDS, (int(v) for v in buf)))

    def profile_timeline(self) -> np.ndarray:
        """Per-op event clocks of a three-level delete server (profiling
        handles): ops kTlFirst.. of the first hold, 32 events each (see
        bh_heap.cuh tl())."""
        base, ops = 64 + 4 * 4096, 64
        buf = (C.c_uint64 * (base + ops * 32))()
        _raise(L.lib().bh_profile(self._h, buf, base + ops * 32, 0))
        return np.frombuffer(buf, dtype=np.uint64)[base:].reshape(ops, 32).copy()

    def profile_levels(self) -> dict:
        """Per-level BU climb profile (profiling handles), indexed by the
        level of the parent a climb step claims (0 = root): steps, mean
        parent-claim wait and mean claim-to-release time in SM cycles (see
        bh_heap.cuh pf_lv)."""
        base = 64 + 4 * 4096 + 64 * 32
        buf = (C.c_uint64 * (base + 3 * 32))()
        _raise(L.lib().bh_profile(self._h, buf, base + 3 * 32, 0))
        a = np.frombuffer(buf, dtype=np.uint64)[base:].reshape(3, 32).astype(np.float64)
        n = a[0]
        with np.errstate(invalid="ignore", divide="ignore"):
            return {"steps": n.astype(np.int64), "claim_cycles": np.where(n > 0, a[1] / n, 0.0),
                    "hold_cycles": np.where(n > 0, a[2] / n, 0.0)}

    def info(self) -> dict:
        k, kb, mn, tpc, mc = (C.c_uint32() for _ in range(5))
        sc = C.c_uint64()
        var = C.c_int()
        _raise(L.lib().bh_info(self._h, C.byref(k), C.byref(kb), C.byref(sc), C.byref(mn),
                               C.byref(var), C.byref(tpc), C.byref(mc)))
        return {"k": k.value, "key_bits": kb.value, "slot_count": sc.value, "max_nodes": mn.value,
                "variant": var.value, "threads_per_cta": tpc.value, "max_ctas": mc.value}

    @property
    def variant(self) -> Variant:
        return self._variant

    def node_capacity(self) -> int:
        return self._k

    def max_nodes(self) -> int:
        return self._max_nodes


OP_DTYPE = np.dtype([("kind", np.uint32), ("len", np.uint32), ("offset", np.uint64)])
EVENT_DTYPE = np.dtype([("ts", np.uint64), ("op", np.uint32), ("kind", np.uint16),
                        ("pad", np.uint16), ("node", np.uint64)])


def make_ops(kinds: Sequence[int], lens: Sequence[int], offsets: Sequence[int]) -> np.ndarray:
    ops = np.empty(len(kinds), dtype=OP_DTYPE)
    ops["kind"] = kinds
    ops["len"] = lens
    ops["offset"] = offsets
    return ops


def phase_ops(kind: int, n_keys: int, k: int) -> np.ndarray:
    """The benchmark's phase plan: inserts of consecutive k-chunks, or
    ceil(n/k) deletes writing consecutive k-wide slots."""
    n_ops = (n_keys + k - 1) // k
    at = np.arange(n_ops, dtype=np.uint64) * np.uint64(k)
    if kind == L.BH_OP_INSERT:
        lens = np.minimum(np.uint64(k), np.uint64(n_keys) - at).astype(np.uint32)
        return make_ops(np.zeros(n_ops, np.uint32), lens, at)
    return make_ops(np.ones(n_ops, np.uint32), np.zeros(n_ops, np.uint32), at)


# ------------------------------------------------- batch primitives ------
def slot_for_rank(rank: int) -> int:
    """proj/include/batchheap/bitrev.hpp:29-33."""
    return int(L.lib().bh_slot_for_rank(rank))


def bit_reverse(x: int, bits: int) -> int:
    return int(L.lib().bh_bit_reverse(x, bits))


def path_to_slot(slot: int):
    """proj/include/batchheap/bitrev.hpp:36-42."""
    path = []
    while slot >= 1:
        path.append(slot)
        slot //= 2
    return path[::-1]


def level_of_rank(rank: int) -> int:
    return rank.bit_length() - 1


def generate_keys(n: int, seed: int = 1, order: int = 0, key_bits: int = 64) -> np.ndarray:
    """generate_keys (proj/src/workload.cpp:162-180), host C++ generator."""
    out = np.empty(max(n, 1), dtype=_key_dtype(key_bits))
    _raise(L.lib().bh_generate_keys(order, n, seed, key_bits, out.ctypes.data_as(C.c_void_p)))
    return out[:n]


def sort_batches_device(keys_ptr: int, k: int, rows: int, key_bits: int, lens_ptr: int = 0,
                        stream: int = 0) -> None:
    """sort_batch on device rows (stride k) in place."""
    _raise(L.lib().bh_sort_batches(key_bits, k, keys_ptr, lens_ptr or None, rows, stream or None))


def merge_split_device(a_ptr: int, b_ptr: int, hi_ptr: int, lo_ptr: int, k: int, pairs: int,
                       key_bits: int, stream: int = 0) -> None:
    """merge_and_sort on device row pairs."""
    _raise(L.lib().bh_merge_split(key_bits, k, a_ptr, b_ptr, hi_ptr, lo_ptr, pairs, stream or None))
