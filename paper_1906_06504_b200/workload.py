"""The reference's benchmark harness on the device heap
(proj/include/batchheap/bench.hpp, proj/src/bench.cpp,
proj/include/batchheap/workload.hpp).

``WorkloadSpec`` / ``BenchRow`` / ``run_workload`` / ``run_sweep`` /
``write_csv`` keep the reference's fields, semantics and CSV columns, so GPU
and CPU rows compare column for column:

* keys: ``generate_keys(order, total_keys, seed)``; batches: the reference's
  ``plan_batches`` (``bh_plan_batches``: per-worker shares, full_batch_pct);
  ``initial_levels`` complete levels pre-inserted from
  ``generate_keys(Random, ..., seed ^ 0x5851f42d4c957f2d)``, then counters
  reset (bench.cpp:56-72);
* ``InsertAllThenDeleteAll``: every batch inserted, then deleteMin until all
  keys are out; ``InsDelPairs``: per batch an insert followed by a deleteMin
  (bench.cpp:75-115).  The reference's ``workers`` threads become one bulk
  run over ``ctas`` persistent CTAs (0 = all co-resident); ``workers`` still
  shapes the batch plan and the op order (worker-major);
* every timed run is preceded by a correctness pass on the same seed
  (quiescent invariants + multiset conservation, bench.cpp:127-147); the
  time is device time of the op launches (CUDA events), the reference's is
  wall time around its op loop.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import Iterable, List, Optional, TextIO

import numpy as np

from . import _lib as L
from .heap import GeneralizedHeap, HeapCounters, HeapOptions, Variant, _raise, generate_keys, make_ops


class KeyOrder(enum.IntEnum):  # workload.hpp
    Random = 0
    Ascend = 1
    Descend = 2


class OpPattern(enum.IntEnum):  # workload.hpp
    InsertAllThenDeleteAll = 0
    InsDelPairs = 1


def key_order_name(order: KeyOrder) -> str:  # workload.cpp:149-156
    return {KeyOrder.Random: "random", KeyOrder.Ascend: "ascend", KeyOrder.Descend: "descend"}[KeyOrder(order)]


def op_pattern_name(pattern: OpPattern) -> str:  # workload.cpp:158-160
    return "insall" if OpPattern(pattern) == OpPattern.InsertAllThenDeleteAll else "pairs"


def variant_name(v: Variant) -> str:  # history.hpp:25-27
    return "td" if Variant(v) == Variant.TD else "bu"


@dataclasses.dataclass
class WorkloadSpec:
    """WorkloadSpec (bench.hpp:14-25) plus the device CTA count."""
    variant: Variant = Variant.TD
    k: int = 64
    workers: int = 4
    total_keys: int = 1_000_000
    key_order: KeyOrder = KeyOrder.Random
    op_pattern: OpPattern = OpPattern.InsertAllThenDeleteAll
    initial_levels: int = 0
    full_batch_pct: int = 100
    seed: int = 1
    options: HeapOptions = dataclasses.field(default_factory=HeapOptions)
    ctas: int = 0


@dataclasses.dataclass
class BenchRow:
    """BenchRow (bench.hpp:27-34)."""
    spec: WorkloadSpec
    wall_seconds: float = 0.0
    ops: int = 0
    ops_per_second: float = 0.0
    mean_nodes_traversed: float = 0.0
    counters: Optional[HeapCounters] = None


def plan_batches(spec: WorkloadSpec) -> np.ndarray:
    """Batch lengths of plan_batches (bench.cpp:21-47), worker-major."""
    n = C.c_uint64(0)
    lib = L.lib()
    _raise(lib.bh_plan_batches(spec.k, spec.total_keys, spec.workers, spec.full_batch_pct, spec.seed, None, None,
                               0, C.byref(n)))
    lens = np.empty(max(n.value, 1), dtype=np.uint32)
    _raise(lib.bh_plan_batches(spec.k, spec.total_keys, spec.workers, spec.full_batch_pct, spec.seed,
                               lens.ctypes.data_as(C.c_void_p), None, lens.size, C.byref(n)))
    return lens[:n.value]


def _ops(spec: WorkloadSpec, lens: np.ndarray, n_keys_total: int):
    offs = np.concatenate([[0], np.cumsum(lens, dtype=np.uint64)[:-1]]).astype(np.uint64)
    nb = lens.size
    if spec.op_pattern == OpPattern.InsertAllThenDeleteAll:
        n_del = (n_keys_total + spec.k - 1) // spec.k + 1
        ins = make_ops(np.zeros(nb, np.uint32), lens, offs)
        dels = make_ops(np.ones(n_del, np.uint32), np.zeros(n_del, np.uint32),
                        np.arange(n_del, dtype=np.uint64) * spec.k)
        return [ins, dels], n_del * spec.k
    kinds = np.tile(np.array([0, 1], np.uint32), nb)
    ln = np.empty(2 * nb, np.uint32)
    ln[0::2], ln[1::2] = lens, 0
    of = np.empty(2 * nb, np.uint64)
    of[0::2], of[1::2] = offs, np.arange(nb, dtype=np.uint64) * spec.k
    return [make_ops(kinds, ln, of)], nb * spec.k


def _run_once(spec: WorkloadSpec, verify: bool, device: int):
    import torch

    keys = generate_keys(spec.total_keys, spec.seed, order=int(spec.key_order), key_bits=64)
    seed_nodes = (1 << spec.initial_levels) - 1 if spec.initial_levels else 0
    max_nodes = seed_nodes + spec.total_keys // spec.k + spec.workers + 2 + 64
    heap = GeneralizedHeap(spec.variant, spec.k, max_nodes, spec.options, key_bits=64, device=device)
    try:
        seed_keys = generate_keys(seed_nodes * spec.k, spec.seed ^ 0x5851F42D4C957F2D, key_bits=64)
        if seed_nodes:
            heap.run_ops(make_ops(np.zeros(seed_nodes, np.uint32), np.full(seed_nodes, spec.k, np.uint32),
                                  np.arange(seed_nodes, dtype=np.uint64) * spec.k), seed_keys, 0, ctas=spec.ctas)
        heap.reset_counters()
        lens = plan_batches(spec)
        op_lists, out_len = _ops(spec, lens, spec.total_keys + seed_keys.size)
        dev = torch.device("cuda", device)
        pool = torch.from_numpy(keys.view(np.int64)).to(dev)
        out = torch.empty(max(out_len, 1), dtype=torch.int64, device=dev)
        d_ops = [torch.from_numpy(o.view(np.uint8)).to(dev) for o in op_lists]
        st = [torch.zeros(len(o), dtype=torch.int32, device=dev) for o in op_lists]
        lens_d = [torch.zeros(len(o), dtype=torch.int32, device=dev) for o in op_lists]
        s = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(s)
        for o, do, sd, ld in zip(op_lists, d_ops, st, lens_d):
            heap.run_ops_ptr(do.data_ptr(), len(o), pool.data_ptr(), out.data_ptr(), sd.data_ptr(), ld.data_ptr(),
                             0, ctas=spec.ctas, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize(dev)
        seconds = e0.elapsed_time(e1) / 1e3
        counters = heap.counters()
        ok, detail = True, ""
        if verify:
            rep = heap.check_invariants()
            if not rep.ok:
                return seconds, counters, False, rep.detail
            outs = out.cpu().numpy().view(np.uint64)
            deleted = []
            for o, ld in zip(op_lists, lens_d):
                ln = ld.cpu().numpy()
                for i in np.nonzero(o["kind"] == 1)[0]:
                    at = int(o["offset"][i])
                    deleted.append(outs[at:at + int(ln[i])])
            acc = np.sort(np.concatenate(deleted + [heap.collect_resident().astype(np.uint64)]))
            ins = np.sort(np.concatenate([keys.astype(np.uint64), seed_keys.astype(np.uint64)]))
            if not np.array_equal(acc, ins):
                ok, detail = False, "multiset conservation failed"
        return seconds, counters, ok, detail
    finally:
        heap.close()


def run_workload(spec: WorkloadSpec, device: int = 0) -> BenchRow:
    """run_workload (bench.cpp:167-184): a verified pass, then a timed one."""
    _, _, ok, detail = _run_once(spec, True, device)
    if not ok:
        raise RuntimeError(f"correctness pass failed for {variant_name(spec.variant)} k={spec.k} "
                           f"workers={spec.workers} keys={spec.total_keys} seed={spec.seed}: {detail}")
    seconds, c, _, _ = _run_once(spec, False, device)
    ops = c.inserts + c.deletes
    return BenchRow(spec, seconds, ops, ops / seconds if seconds > 0 else 0.0,
                    c.propagation_node_visits / ops if ops else 0.0, c)


def run_sweep(grid: Iterable[WorkloadSpec], device: int = 0) -> List[BenchRow]:  # bench.cpp:186-192
    return [run_workload(s, device) for s in grid]


CSV_HEADER = ("variant,k,workers,total_keys,key_order,op_pattern,initial_levels,full_batch_pct,seed,wall_seconds,"
              "ops,throughput_ops_s,mean_nodes_traversed,merge_count,early_stop_count,max_partial_occupancy")


def _num(x: float) -> str:
    return f"{x:g}"  # std::ostream default formatting (6 significant digits)


def write_csv(out: TextIO, rows: Iterable[BenchRow]) -> None:
    """write_csv (bench.cpp:194-210), same columns and order."""
    out.write(CSV_HEADER + "\n")
    for r in rows:
        s = r.spec
        out.write(",".join([variant_name(s.variant), str(s.k), str(s.workers), str(s.total_keys),
                            key_order_name(s.key_order), op_pattern_name(s.op_pattern), str(s.initial_levels),
                            str(s.full_batch_pct), str(s.seed), _num(r.wall_seconds), str(r.ops),
                            _num(r.ops_per_second), _num(r.mean_nodes_traversed), str(r.counters.merges),
                            str(r.counters.early_stops), str(r.counters.max_partial_len)]) + "\n")
