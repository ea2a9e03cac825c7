import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant
from test_gpu_bulk import mixed_ops
for k in (4, 64):
    rng = np.random.default_rng(k)
    ops, pool, out_len, _ = mixed_ops(rng, 600, k, 20, 1 << 24)
    res = []
    for flags in (0, 0x1000):
        heap = GeneralizedHeap(Variant.BU, k, 700, debug_flags=flags)
        r = heap.run_ops(ops, pool, out_len, ctas=1)
        keys, part, states = heap.dump()
        res.append((keys.copy(), part.copy(), heap.counters().__dict__, r.out.copy(), r.status.copy(), heap.check_invariants().ok))
    a, b = res
    print(k, "keys eq", np.array_equal(a[0], b[0]), "part eq", np.array_equal(a[1], b[1]), "out eq", np.array_equal(a[3], b[3]),
          "status eq", np.array_equal(a[4], b[4]), "inv", a[5], b[5])
    print(" counters gated", a[2]); print(" counters ref  ", b[2])
    # oracle sequential replay
    orc = O.SeqHeap(1, k, 700, True)
    for i, o in enumerate(ops):
        if o["kind"] == 0:
            orc.insert(pool[o["offset"]:o["offset"] + o["len"]])
        else:
            orc.delete_min()
    ko, po = orc.dump()
    print(" oracle keys eq gated", np.array_equal(a[0].astype(np.uint64), ko), "ref", np.array_equal(b[0].astype(np.uint64), ko))
    print(" oracle counters", orc.counters())
