"""Diagnostic: where do keys go wrong in a drain (tooling)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops
log2n = int(sys.argv[1]); flags = int(sys.argv[2], 0); k = 1024
n = 1 << log2n
keys = O.generate_keys(n, 11)
want = O.sort_u64(keys)
for rep in range(3):
    heap = GeneralizedHeap(Variant.BU, k, n // k + 64, key_bits=32, debug_flags=flags)
    heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
    d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
    order = np.argsort(d.seq, kind="stable")
    out = d.out.reshape(n // k, k)[order].astype(np.uint64)
    flat = out.reshape(-1)
    if np.array_equal(flat, want):
        print("ok"); continue
    u, c = np.unique(flat, return_counts=True)
    dup = u[c > 1]
    missing = np.setdiff1d(want, flat)
    print(f"rep {rep}: dups={len(dup)} (sentinels {int(np.sum(flat == 0xFFFFFFFF))}) missing={len(missing)} resident_after={heap.peek_stats().key_count}")
    # first unsorted batch
    for i in range(n // k):
        b = out[i]
        if not np.all(b[:-1] <= b[1:]):
            print("  batch", i, "not sorted"); break
        if i and out[i - 1][-1] > b[0]:
            print(f"  batch {i} overlaps previous: prev max {out[i-1][-1]} this min {b[0]}"); break
    if len(dup):
        dv = dup[0]
        where = np.argwhere(out == dv)
        print("  dup key", dv, "in batches", where[:, 0].tolist(), "positions", where[:, 1].tolist())
    if len(missing):
        print("  missing sample", missing[:5], "rank in want", np.searchsorted(want, missing[:5]))
    print("  invariants:", heap.check_invariants().ok, heap.check_invariants().detail[:200])
