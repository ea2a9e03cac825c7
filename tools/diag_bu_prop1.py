"""Hunt the rare BU quiescent property-1 violation: run recorded BU mixed
workloads at k=1 until check_invariants fails, then dump the violating
slot, its parent, and every recorded lock span on them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from oracle import lincheck as LC
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import _recorded_history, mixed_ops

found = 0
for trial in range(300):
    k = 1 if trial % 2 == 0 else 2
    rng = np.random.default_rng(trial)
    ops, pool, out_len, _ = mixed_ops(rng, 4000, k, 20, 1 << 40)
    heap = GeneralizedHeap(Variant.BU, k, 4100, record=True)
    r = heap.run_ops(ops, pool, out_len, ctas=128)
    rep = heap.check_invariants()
    if rep.ok:
        continue
    found += 1
    print(f"trial {trial} k={k}: {rep.detail}")
    keys, part, states = heap.dump()
    nodes = heap.peek_stats().node_count
    bad = int(rep.detail.split("first ")[1].split(":")[0])
    par = bad // 2
    print(f"  nodes={nodes} slot {bad} keys={keys[bad-1].tolist()} parent {par} keys={keys[par-1].tolist()}")
    hist = _recorded_history(heap, ops, r, pool)
    spans = []
    for op in hist:
        for s in op.locks:
            if s.node in (bad, par, 2 * bad, 2 * bad + 1):
                spans.append((s.acquire_ts, s.release_ts, s.node, "ins" if op.op == 0 else "del", op.opid,
                              op.keys[:2]))
    spans.sort()
    for sp in spans[-40:]:
        print("   ", sp)
    if found >= 3:
        break
print("violations found:", found)
