"""ctypes front-end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker.  The
product package (``paper_1906_06504_b200``) never imports it.

Two libraries sit behind it:

* ``oracle/_build/libbhoracle.so`` -- the plain-C restatement in
  ``oracle/bh_oracle.c`` (always built by ``__graft_entry__.build()``).
* ``oracle/_ref/libbatchheap_ref.so`` -- the reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` (optional; present when
  the reference was available at build time, and shipped to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libbhoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbatchheap_ref.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")

OK, E_CONFIG, E_CAPACITY, E_EMPTY, E_INVALID_KEY = 0, 1, 2, 3, 4
TD, BU = 0, 1
RANDOM, ASCEND, DESCEND = 0, 1, 2


class _Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "inserts", "deletes", "merges", "elided_merges", "early_stops",
        "propagation_node_visits", "coop_handoffs", "max_partial_len")]


def _load_oracle():
    if not os.path.exists(ORACLE_SO):
        raise RuntimeError(f"oracle library missing: {ORACLE_SO} (run make -C oracle)")
    lib = C.CDLL(ORACLE_SO)
    lib.orc_generate_keys.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _u64p]
    lib.orc_sort_u64.argtypes = [_u64p, C.c_uint64]
    lib.orc_merge_sorted.argtypes = [_u64p, C.c_uint64, _u64p, C.c_uint64, _u64p]
    lib.orc_needs_merge.argtypes = [_u64p, C.c_uint64, _u64p, C.c_uint64]
    lib.orc_bit_reverse.argtypes = [C.c_uint64, C.c_uint]
    lib.orc_bit_reverse.restype = C.c_uint64
    lib.orc_slot_for_rank.argtypes = [C.c_uint64]
    lib.orc_slot_for_rank.restype = C.c_uint64
    lib.orc_heap_create.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32]
    lib.orc_heap_create.restype = C.c_void_p
    lib.orc_heap_destroy.argtypes = [C.c_void_p]
    lib.orc_heap_insert.argtypes = [C.c_void_p, _u64p, C.c_uint32]
    lib.orc_heap_delete.argtypes = [C.c_void_p, _u64p, C.POINTER(C.c_uint32)]
    lib.orc_heap_slot_count.argtypes = [C.c_void_p]
    lib.orc_heap_slot_count.restype = C.c_uint64
    lib.orc_heap_node_count.argtypes = [C.c_void_p]
    lib.orc_heap_node_count.restype = C.c_uint64
    lib.orc_heap_partial_len.argtypes = [C.c_void_p]
    lib.orc_heap_partial_len.restype = C.c_uint32
    lib.orc_heap_dump.argtypes = [C.c_void_p, _u64p, _u64p]
    lib.orc_heap_counters.argtypes = [C.c_void_p, C.POINTER(_Counters)]
    lib.orc_grid_graph_edges.argtypes = [C.c_uint32, C.c_uint32]
    lib.orc_grid_graph_edges.restype = C.c_uint64
    lib.orc_grid_graph.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u64p, _u32p, _u32p]
    lib.orc_dijkstra.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_uint32, _u64p]
    lib.orc_generate_knapsack.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, _u32p, _u32p]
    lib.orc_generate_knapsack.restype = C.c_uint64
    lib.orc_knapsack_dp.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64]
    lib.orc_knapsack_dp.restype = C.c_uint64
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load_oracle()
    return _lib


# ------------------------------------------------------------------ keys --
def generate_keys(n: int, seed: int = 1, order: int = RANDOM) -> np.ndarray:
    """generate_keys (proj/src/workload.cpp:162-180) as uint64."""
    out = np.empty(n, dtype=np.uint64)
    lib().orc_generate_keys(order, n, seed, out)
    return out


def sort_u64(a: np.ndarray) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.uint64).copy()
    lib().orc_sort_u64(out, out.size)
    return out


def merge_sorted(a, b) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty(a.size + b.size, dtype=np.uint64)
    lib().orc_merge_sorted(a, a.size, b, b.size, out)
    return out


def merge_and_sort(a, b, k: int):
    """merge_and_sort (proj/src/batch.cpp:32-42)."""
    m = merge_sorted(a, b)
    cut = min(k, m.size)
    return m[:cut], m[cut:]


def needs_merge(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    return bool(lib().orc_needs_merge(a, a.size, b, b.size))


def bit_reverse(x: int, bits: int) -> int:
    return int(lib().orc_bit_reverse(x, bits))


def slot_for_rank(rank: int) -> int:
    return int(lib().orc_slot_for_rank(rank))


def path_to_slot(slot: int):
    path = []
    while slot >= 1:
        path.append(slot)
        slot //= 2
    return path[::-1]


def checksums(sorted_keys: np.ndarray):
    """(sum, xor, polynomial hash h = h*1000003 + key mod 2^64) -- the
    fingerprints of SURVEY.md Appendix B."""
    s = int(sorted_keys.astype(np.uint64).sum(dtype=np.uint64))
    x = int(np.bitwise_xor.reduce(sorted_keys.astype(np.uint64))) if sorted_keys.size else 0
    h = 0
    mask = (1 << 64) - 1
    # vectorised Horner in chunks: h_{i+1} = h_i*P + k_i
    P = 1000003
    keys = sorted_keys.astype(np.uint64)
    chunk = 1 << 16
    # powers of P mod 2^64 for a chunk
    pw = np.empty(chunk, dtype=np.uint64)
    acc = 1
    for i in range(chunk):
        pw[chunk - 1 - i] = acc
        acc = (acc * P) & mask
    p_chunk = acc
    with np.errstate(over="ignore"):
        for at in range(0, keys.size, chunk):
            part = keys[at:at + chunk]
            m = part.size
            if m == chunk:
                contrib = int((part * pw).sum(dtype=np.uint64))
                h = (h * p_chunk + contrib) & mask
            else:
                for v in part.tolist():
                    h = (h * P + v) & mask
    return s, x, h


# ------------------------------------------------------------ seq heap ----
class SeqHeap:
    """Sequential execution of GeneralizedHeap (oracle/bh_oracle.c)."""

    def __init__(self, variant: int, k: int, max_nodes: int, elide: bool = True, key_bits: int = 64):
        self.k = k
        self.key_bits = key_bits
        self._h = lib().orc_heap_create(variant, k, max_nodes, int(elide), key_bits)
        if not self._h:
            raise ValueError("bad heap config")
        self.slot_count = int(lib().orc_heap_slot_count(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_heap_destroy(self._h)
            self._h = None

    def insert(self, items) -> int:
        a = np.ascontiguousarray(items, dtype=np.uint64)
        return lib().orc_heap_insert(self._h, a, a.size)

    def delete_min(self):
        out = np.empty(self.k, dtype=np.uint64)
        n = C.c_uint32(0)
        st = lib().orc_heap_delete(self._h, out, C.byref(n))
        return st, out[:n.value].copy()

    @property
    def node_count(self) -> int:
        return int(lib().orc_heap_node_count(self._h))

    @property
    def partial_len(self) -> int:
        return int(lib().orc_heap_partial_len(self._h))

    def dump(self):
        keys = np.empty(self.slot_count * self.k, dtype=np.uint64)
        part = np.empty(self.k, dtype=np.uint64)
        lib().orc_heap_dump(self._h, keys, part)
        return keys.reshape(self.slot_count, self.k), part[:self.partial_len].copy()

    def counters(self) -> dict:
        c = _Counters()
        lib().orc_heap_counters(self._h, C.byref(c))
        return {n: int(getattr(c, n)) for n, _ in _Counters._fields_}


# ------------------------------------------------------------ apps --------
def grid_graph(rows: int, cols: int, seed: int):
    n = rows * cols
    m = int(lib().orc_grid_graph_edges(rows, cols))
    off = np.empty(n + 1, dtype=np.uint64)
    nbr = np.empty(m, dtype=np.uint32)
    w = np.empty(m, dtype=np.uint32)
    lib().orc_grid_graph(rows, cols, seed, off, nbr, w)
    return off, nbr, w


def dijkstra(offsets, nbr, wgt, source: int) -> np.ndarray:
    n = offsets.size - 1
    dist = np.empty(n, dtype=np.uint64)
    lib().orc_dijkstra(n, offsets, nbr, wgt, source, dist)
    return dist


def generate_knapsack(kind: int, n: int, rng_range: int, seed: int):
    w = np.empty(n, dtype=np.uint32)
    b = np.empty(n, dtype=np.uint32)
    cap = int(lib().orc_generate_knapsack(kind, n, rng_range, seed, w, b))
    return w, b, cap


def knapsack_dp(w, b, cap: int) -> int:
    return int(lib().orc_knapsack_dp(w.size, w, b, cap))


# -------------------------------------------------- reference library -----
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The unmodified reference library (oracle/_ref), or raise."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference library not built: {REF_SO}")
        r = C.CDLL(REF_SO)
        r.ref_last_error.restype = C.c_char_p
        r.ref_generate_keys.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _u64p]
        r.ref_heap_create.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_int]
        r.ref_heap_create.restype = C.c_void_p
        r.ref_heap_destroy.argtypes = [C.c_void_p]
        r.ref_heap_insert.argtypes = [C.c_void_p, _u64p, C.c_uint32]
        r.ref_heap_delete.argtypes = [C.c_void_p, _u64p, C.POINTER(C.c_uint32)]
        r.ref_heap_peek.argtypes = [C.c_void_p, _u64p]
        r.ref_heap_counters.argtypes = [C.c_void_p, _u64p]
        r.ref_heap_collect.argtypes = [C.c_void_p, _u64p, C.c_uint64]
        r.ref_heap_collect.restype = C.c_uint64
        r.ref_heap_check.argtypes = [C.c_void_p]
        r.ref_phase.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
        r.ref_run_workload.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_int,
                                       C.c_uint32, C.c_uint32, C.c_uint64,
                                       np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
        r.ref_grid_dijkstra.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, _u64p]
        r.ref_grid_sssp.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                    C.c_uint32, _u64p, C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_double)]
        r.ref_generate_knapsack.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, _u32p, _u32p]
        r.ref_generate_knapsack.restype = C.c_uint64
        r.ref_knapsack_dp.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64]
        r.ref_knapsack_dp.restype = C.c_uint64
        r.ref_knapsack_bb.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                      C.c_uint32, _u64p, C.POINTER(C.c_double)]
        _ref = r
    return _ref


def ref_phase(variant: int, k: int, n_keys: int, workers: int, seed: int = 1, verify: bool = False):
    """Time the reference GeneralizedHeap: returns (insert_s, delete_s)."""
    t = np.zeros(2, dtype=np.float64)
    st = ref().ref_phase(variant, k, n_keys, workers, seed, int(verify), t)
    if st != 0:
        raise RuntimeError(f"ref_phase failed ({st}): {ref().ref_last_error().decode()}")
    return float(t[0]), float(t[1])


def ref_knapsack_bb_subprocess(kind: int, n: int, rng_range: int, seed: int, workers: int = 2,
                               gc_threshold: int = 1 << 16, k: int = 32, timeout: float = 120.0) -> dict:
    """The reference's knapsack_bb in a child process (an arena exhaustion
    terminates the process, knapsack.cpp:136-154): {best, explored, gc,
    seconds} or {error}."""
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {os.path.dirname(HERE)!r});"
            "import ctypes as C, numpy as np; from oracle import oracle as O;"
            "o = np.zeros(3, np.uint64); t = C.c_double();"
            f"st = O.ref().ref_knapsack_bb({kind}, {n}, {rng_range}, {seed}, {workers}, {gc_threshold}, {k}, o,"
            " C.byref(t));"
            "print(st, int(o[0]), int(o[1]), int(o[2]), t.value)")
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": f"timeout {timeout}s"}
    if r.returncode != 0 or not r.stdout.strip():
        return {"error": f"terminated (rc {r.returncode}): {r.stderr.strip()[-160:]}"}
    st, best, explored, gc, secs = r.stdout.split()
    if int(st) != 0:
        return {"error": f"status {st}"}
    return {"best": int(best), "explored": int(explored), "gc": int(gc), "seconds": float(secs)}


REF_HISTCHECK = os.path.join(HERE, "_ref", "ref_histcheck")


def ref_history_check(text: str, variant: int, k: int) -> dict:
    """The reference's History::parse + check_td/check_bu (+ overlap windows
    for BU, + check_exhaustive for <= 16 ops) on a history in its text
    format, via oracle/_ref/ref_histcheck (a separate process)."""
    import subprocess
    r = subprocess.run([REF_HISTCHECK, str(variant), str(k)], input=text, capture_output=True, text=True,
                       timeout=600)
    if r.returncode != 0:
        return {"error": r.stderr.strip()}
    p, o, e, n = (int(x) for x in r.stdout.split())
    return {"pass": bool(p), "overlap_ok": bool(o), "exhaustive": e, "ops": n, "detail": r.stderr.strip()}


class RefHeap:
    """The reference GeneralizedHeap behind ctypes (for cross-checks)."""

    def __init__(self, variant: int, k: int, max_nodes: int, elide: bool = True):
        self.k = k
        self._h = ref().ref_heap_create(variant, k, max_nodes, int(elide))
        if not self._h:
            raise ValueError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            ref().ref_heap_destroy(self._h)
            self._h = None

    def insert(self, items) -> int:
        a = np.ascontiguousarray(items, dtype=np.uint64)
        return ref().ref_heap_insert(self._h, a, a.size)

    def delete_min(self):
        out = np.empty(self.k, dtype=np.uint64)
        n = C.c_uint32(0)
        st = ref().ref_heap_delete(self._h, out, C.byref(n))
        return st, out[:n.value].copy()

    def counters(self) -> dict:
        o = np.zeros(8, dtype=np.uint64)
        ref().ref_heap_counters(self._h, o)
        return dict(zip((n for n, _ in _Counters._fields_), (int(v) for v in o)))

    def peek(self):
        o = np.zeros(4, dtype=np.uint64)
        ref().ref_heap_peek(self._h, o)
        return tuple(int(v) for v in o)
