"""Per-op timeline of the two-level delete server (tooling): one 2^22-key
(or --log2n) phase-separated run at K=1024 with profiling, then the event
clocks of served ops 1000-1015 relative to each op's start (SM cycles)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops

NAMES = {0: "start", 1: "pub flushed", 2: "looked up", 3: "refill done", 4: "H0+lo0 done", 5: "claims done",
         6: "C at split bar", 7: "r1", 8: "r2", 9: "r3", 10: "loop barrier"}
ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=22)
ap.add_argument("--ops", type=int, default=6)
a = ap.parse_args()
n = 1 << a.log2n
k = 1024
keys = O.generate_keys(n, 1)
heap = GeneralizedHeap(Variant.BU, k, n // k + 64, key_bits=32, profile=True)
heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
heap.profile(reset=True)
heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
tlm = heap.profile_timeline().astype(np.int64)
durs = []
for i in range(min(a.ops, 16)):
    row = tlm[i]
    t0 = row[0]
    print(f"op {1000 + i}: " + ", ".join(f"{NAMES[e]} {int(row[e] - t0):+d}" for e in sorted(NAMES, key=lambda e: row[e]) if row[e]) +
          "")
tlm = tlm[:16]
starts = tlm[:, 0]
d = np.diff(starts[starts > 0])
print("op period cycles: median", int(np.median(d)), "mean", int(d.mean()))
for e in sorted(NAMES):
    rel = tlm[1:, e] - tlm[1:, 0]
    print(f"  {NAMES[e]:14s} median {int(np.median(rel)):+6d}")
