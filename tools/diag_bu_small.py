"""Small BU histories: when the constructive check_bu fails, is the history
still linearizable (exhaustive search)?  Prints one non-linearizable
history in full if found."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from oracle import lincheck as LC
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import _recorded_history, mixed_ops

for variant in (Variant.BU, Variant.TD):
    for key_hi in (1 << 40, 12):
        c_fail = e_fail = rep_fail = 0
        shown = False
        for trial in range(1500):
            rng = np.random.default_rng(9000 + trial)
            ops, pool, out_len, _ = mixed_ops(rng, 16, 2, 30, key_hi)
            heap = GeneralizedHeap(variant, 2, 64, record=True)
            r = heap.run_ops(ops, pool, out_len, ctas=16)
            hist = _recorded_history(heap, ops, r, pool)
            strict = LC.check_td(hist, 2) if variant == Variant.TD else LC.check_bu(hist, 2)
            if strict.passed:
                continue
            c_fail += 1
            if variant == Variant.BU and not LC.check_bu_repaired(hist, 2).passed:
                rep_fail += 1
            ex = LC.check_exhaustive(hist, 2)
            if not ex.passed:
                e_fail += 1
                if not shown:
                    shown = True
                    print("NON-LINEARIZABLE history (variant %s):" % variant.name)
                    for op in sorted(hist, key=lambda o: o.invoke_ts):
                        print(f"  {'ins' if op.op == 0 else 'del'} #{op.opid} keys={op.keys} "
                              f"inv={op.invoke_ts} res={op.respond_ts} acR={op.root_acquire_ts} "
                              f"reR={op.root_release_ts} acL={op.last_acquire_ts} reL={op.last_release_ts} "
                              f"locks={[(s.node, s.acquire_ts, s.release_ts) for s in op.locks]}")
        print(f"{variant.name} key_hi={key_hi}: constructive-fail {c_fail}/1500, repaired-fail {rep_fail}, "
              f"exhaustive-fail {e_fail}", flush=True)
