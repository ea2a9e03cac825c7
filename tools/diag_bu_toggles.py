"""Which protocol reordering (if any) causes the rare BU quiescent
property-1 violation?  Many k=1/k=2 mixed runs per toggle, no recording."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import mixed_ops

RUNS = int(sys.argv[1]) if len(sys.argv) > 1 else 60
TOGGLES = {"none": 0, "seq_refill": 0x100, "write_under_root": 0x200, "serial_lanes": 0x400,
           "all": 0x700}
cases = []
for trial in range(RUNS):
    k = 1 if trial % 2 == 0 else 2
    rng = np.random.default_rng(trial)
    cases.append((k,) + mixed_ops(rng, 4000, k, 20, 1 << 40)[:3])
for name, dbg in TOGGLES.items():
    bad = 0
    t0 = time.time()
    for k, ops, pool, out_len in cases:
        heap = GeneralizedHeap(Variant.BU, k, 4100, debug_flags=dbg)
        heap.run_ops(ops, pool, out_len, ctas=128)
        bad += not heap.check_invariants().ok
        heap.close()
    print(f"{name:18s} runs {len(cases)} invariant-fail {bad}  ({time.time() - t0:.1f}s)", flush=True)
