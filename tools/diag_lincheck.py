"""Diagnose constructive linearizability checks on recorded device histories:
strict check_bu / check_td vs the repaired BU witness."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from oracle import lincheck as LC
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import _recorded_history, mixed_ops

for variant in (Variant.TD, Variant.BU):
    for key_hi in (12, 1 << 40):
        stats = {"runs": 0, "strict_fail": 0, "repaired_fail": 0, "moved": 0, "mutex_fail": 0, "order_fail": 0}
        for trial in range(20):
            rng = np.random.default_rng(trial * 101 + int(variant) + (key_hi & 0xFF))
            k = 2 if key_hi == 12 else 8
            ops, pool, out_len, _ = mixed_ops(rng, 600, k, 25, key_hi)
            heap = GeneralizedHeap(variant, k, 700, record=True)
            r = heap.run_ops(ops, pool, out_len, ctas=64)
            hist = _recorded_history(heap, ops, r, pool)
            stats["runs"] += 1
            stats["mutex_fail"] += not LC.check_mutual_exclusion(hist)[0]
            stats["order_fail"] += not LC.check_lock_order(hist)[0]
            strict = LC.check_td(hist, k) if variant == Variant.TD else LC.check_bu(hist, k)
            if not strict.passed:
                stats["strict_fail"] += 1
                if variant == Variant.BU:
                    rep = LC.check_bu_repaired(hist, k)
                    if not rep.passed:
                        stats["repaired_fail"] += 1
                        print("  repaired fail:", rep.detail)
                    else:
                        stats["moved"] += int(rep.detail.split()[1])
                else:
                    print("  td strict fail:", strict.detail)
            if not heap.check_invariants().ok:
                print("  invariants broken")
        print(variant.name, key_hi, stats, flush=True)
