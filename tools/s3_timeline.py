"""Per-op timeline of the three-level delete server (tooling): one 2^20-key
(or --log2n) phase-separated run at K=1024 with profiling, then the event
clocks of a few served ops relative to each op's start (SM cycles)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops

NAMES = {8: "A0 merged", 9: "B0 merged", 10: "C0 merged", 11: "W0 rec seen", 12: "W0 done",
         0: "M start", 1: "M r0", 2: "M rf ok", 3: "M r1", 4: "M c3 ok", 5: "M r2", 6: "M r3", 7: "M record",
         21: "M past op bar", 22: "M allocated", 23: "M decided", 13: "W1 go3", 14: "W1 claimed", 15: "RF go", 16: "RF loaded", 17: "RF released"}
ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=22)
ap.add_argument("--ops", type=int, default=6)
a = ap.parse_args()
n = 1 << a.log2n
k = 1024
keys = O.generate_keys(n, 1)
heap = GeneralizedHeap(Variant.BU, k, n // k + 64, key_bits=32, profile=True, debug_flags=0x4000)
heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
heap.profile(reset=True)
heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
tlm = heap.profile_timeline().astype(np.int64)
durs = []
for i in range(min(a.ops, 16)):
    row = tlm[i]
    t0 = row[0]
    print(f"op {1000 + i}: " + ", ".join(f"{NAMES[e]} {int(row[e] - t0):+d}" for e in sorted(NAMES, key=lambda e: row[e]) if row[e]) +
          f" | claim tries {row[18]} refill guess {row[20]}")
tlm = tlm[:16]
starts = tlm[:, 0]
d = np.diff(starts[starts > 0])
print("op period cycles: median", int(np.median(d)), "mean", int(d.mean()))
for e in sorted(NAMES):
    rel = tlm[1:, e] - tlm[1:, 0]
    print(f"  {NAMES[e]:14s} median {int(np.median(rel)):+6d}")
