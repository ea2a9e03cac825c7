"""Stress: repeated insert-all / delete-all drains at one K, checked against
the oracle's sorted stream; prints failures per debug-flag setting
(tooling).  usage: stress_drain.py LOG2N REPS K FLAGS..."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops
log2n, reps, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
flags_list = [int(x, 0) for x in sys.argv[4:]] or [0]
n = 1 << log2n
for variant in (Variant.BU, Variant.TD):
    for flags in flags_list:
        bad = 0
        for rep in range(reps):
            keys = O.generate_keys(n, 100 + rep)
            want = O.sort_u64(keys)
            heap = GeneralizedHeap(variant, k, n // k + 64, key_bits=32, debug_flags=flags)
            heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
            d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
            out = d.out.reshape(-1, k)[np.argsort(d.seq, kind="stable")].reshape(-1).astype(np.uint64)
            bad += not np.array_equal(out, want)
            heap.close()
        print(f"{variant.name} k={k} 2^{log2n} flags={flags:#x}: {bad}/{reps} failed", flush=True)
