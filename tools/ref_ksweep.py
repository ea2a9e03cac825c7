"""The reference heap (oracle/_ref, unmodified sources) on BASELINE config 2's
K sweep: insert-all then deleteMin-all of 2^26 random keys (generate_keys
seed 1), BU, all host cores; phase-split timer.  K=2048 is rejected by the
reference (batch.hpp:34-36)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
w = os.cpu_count()
for k in (256, 512, 1024):
    ti, td = O.ref_phase(1, k, n, w, 1, False)
    print(f"reference BU k={k} workers={w} 2^{n.bit_length() - 1}: insert {ti * 1e3:.1f} ms delete {td * 1e3:.1f} ms "
          f"key-ops/s {2 * n / (ti + td):.3e}", flush=True)
