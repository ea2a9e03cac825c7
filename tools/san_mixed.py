"""Small workload for compute-sanitizer (tooling): K=256 (T=128, so delete
serving and the split schedules run), a phase-separated fill and drain of
2^13 keys, then 400 coin-flip ops with 20% partial inserts, BU and TD, 8
CTAs; checks the drain and the multiset.
    compute-sanitizer --tool racecheck python tools/san_mixed.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, make_ops, phase_ops

k, n = 256, 1 << 13
keys = O.generate_keys(n, 9).astype(np.uint32)
for variant in (Variant.BU, Variant.TD):
    heap = GeneralizedHeap(variant, k, 512, key_bits=32)
    heap.run_ops(phase_ops(0, n, k), keys, 0, ctas=8)
    d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n, ctas=8)
    out = d.out.reshape(-1, k)[np.argsort(d.seq, kind="stable")].reshape(-1).astype(np.uint64)
    assert np.array_equal(out, O.sort_u64(keys)), variant
    rng = np.random.default_rng(3)
    kinds, lens, offs, chunks, at, oat = [], [], [], [], 0, 0
    heap.run_ops(phase_ops(0, n, k), keys, 0, ctas=8)
    for _ in range(400):
        if rng.integers(0, 2) == 0:
            m = k if rng.integers(0, 100) >= 20 else int(rng.integers(1, k))
            chunks.append(rng.integers(0, (1 << 32) - 1, size=m, dtype=np.uint64))
            kinds.append(0); lens.append(m); offs.append(at); at += m
        else:
            kinds.append(1); lens.append(0); offs.append(oat); oat += k
    pool = np.concatenate(chunks).astype(np.uint32)
    ops = make_ops(np.array(kinds, np.uint32), np.array(lens, np.uint32), np.array(offs, np.uint64))
    r = heap.run_ops(ops, pool, oat, ctas=8)
    deleted = np.concatenate([r.out[o["offset"]:o["offset"] + r.lens[i]] for i, o in enumerate(ops) if o["kind"] == 1])
    acc = np.sort(np.concatenate([deleted.astype(np.uint64), heap.collect_resident()]))
    assert np.array_equal(acc, np.sort(np.concatenate([keys, pool]).astype(np.uint64))), variant
    assert heap.check_invariants().ok
    heap.close()
print("san_mixed ok")
