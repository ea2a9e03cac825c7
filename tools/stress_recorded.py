"""Stress of the recorded K=1024 linearizability check (tooling): the
tests/test_gpu_config3.py recorded run (255 seeded nodes, 4096 coin-flip
ops, 20% / 0% partials, all co-resident CTAs, BU and TD) over several
seeds, each through validate, mutual exclusion, lock order, check_td /
check_bu, the JIT witness, invariants and the multiset.
    python tools/stress_recorded.py SEEDS"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from oracle import lincheck as LC
from paper_1906_06504_b200 import GeneralizedHeap, Variant
import test_gpu_config3 as T

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
fails = 0
t0 = time.time()
for variant in (Variant.BU, Variant.TD):
    for pct in (20, 0):
        for s in range(seeds):
            rng = np.random.default_rng(777 + 31 * s + int(variant) + pct)
            seed_nodes = 255
            ops, pool, out_len = T.coin_flip_ops(rng, 4096, 1024, pct, (1 << 32) - 1, seed_nodes, np.uint32,
                                                 tail_deletes=128)
            heap = GeneralizedHeap(variant, 1024, seed_nodes + len(ops) + 8, key_bits=32, record=True, profile=True)
            r = heap.run_ops(ops, pool, out_len)
            served = heap.profile()["del_served"]
            hist = T.recorded_history(heap, ops, r, pool)
            why = LC.validate(hist)
            ok = why is None
            for chk in (LC.check_mutual_exclusion, LC.check_lock_order):
                if ok:
                    ok, why = chk(hist)
            if ok:
                res = LC.check_td(hist, 1024) if variant == Variant.TD else LC.check_bu(hist, 1024)
                ok, why = res.passed, res.detail
            if ok:
                res = LC.check_jit(hist, 1024)
                ok, why = res.passed, res.detail
            if ok:
                rep = heap.check_invariants()
                ok, why = rep.ok, rep.detail
            fails += not ok
            print(f"{variant.name} partial={pct}% seed={s}: {'ok' if ok else 'FAIL ' + str(why)} served={served} "
                  f"refill-overlaps={T.refill_overlaps(hist)} ({time.time() - t0:.0f}s)", flush=True)
            heap.close()
print(f"stress_recorded: {fails} failures", flush=True)
