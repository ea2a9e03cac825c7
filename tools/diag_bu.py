"""Isolate BU invariant failures: mixed concurrent runs with protocol toggles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from oracle import lincheck as LC
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import _recorded_history, mixed_ops

TOGGLES = {"none": 0, "seq_refill": 0x100, "write_under_root": 0x200, "serial_lanes": 0x400,
           "all": 0x700}
for name, dbg in TOGGLES.items():
    inv_bad = ms_bad = lin_bad = 0
    runs = 0
    for trial in range(12):
        rng = np.random.default_rng(trial)
        k = 4 if trial % 2 else 8
        ops, pool, out_len, _ = mixed_ops(rng, 3000, k, 20, 1 << 40)
        heap = GeneralizedHeap(Variant.BU, k, 3100, debug_flags=dbg, record=True)
        r = heap.run_ops(ops, pool, out_len, ctas=128)
        runs += 1
        rep = heap.check_invariants()
        inv_bad += not rep.ok
        deleted = np.concatenate([r.out[o["offset"]:o["offset"] + r.lens[i]]
                                  for i, o in enumerate(ops) if o["kind"] == 1] + [np.zeros(0, np.uint64)])
        acc = np.sort(np.concatenate([deleted.astype(np.uint64), heap.collect_resident()]))
        ms_bad += not np.array_equal(acc, O.sort_u64(pool))
        hist = _recorded_history(heap, ops, r, pool)
        lin_bad += not LC.check_bu(hist, k).passed
    print(f"{name:18s} runs {runs} invariant-fail {inv_bad} multiset-fail {ms_bad} check_bu-fail {lin_bad}",
          flush=True)
