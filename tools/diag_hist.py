import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
from oracle import lincheck as LC
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from paper_1906_06504_b200.history import history_of
from test_gpu_bulk import mixed_ops, _recorded_history
rng = np.random.default_rng(500)
ops, pool, out_len, _ = mixed_ops(rng, 14, 2, 25, 12)
heap = GeneralizedHeap(Variant.TD, 2, 22, record=True)
r = heap.run_ops(ops, pool, out_len, ctas=64)
ev = heap.history_events()
print("status", r.status.tolist())
for i in range(len(ops)):
    e = ev[ev["op"] == i]
    print(i, int(ops[i]["kind"]), [(int(x["ts"]), int(x["kind"]), int(x["node"])) for x in e])
h = history_of(heap, ops, r, pool)
for o in h.ops:
    print(o.opid, o.op, o.invoke_ts, o.root_acquire_ts, o.root_release_ts, o.respond_ts, [(s.node, s.acquire_ts, s.release_ts) for s in o.locks])
