"""Three-level delete server check (tooling): drains and partial drains at
one K with the three-level server (flags 0x4000), the two-level one (0) and
no serving (0x2000); outputs, counters and the heap left behind must agree.
usage: check_serve3.py LOG2N K [REPS]
The server is compiled only into the SERVE3=1 library
(make -C paper_1906_06504_b200/csrc SERVE3=1; BH_LIB=build_var/libbatchheap_b200_serve3.so);
with the shipped library flag 0x4000 falls back to the two-level server and
s3_ops stays 0."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops

log2n, k = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 1 << log2n
fails = 0
for variant in (Variant.BU, Variant.TD):
    for rep in range(reps):
        keys = O.generate_keys(n, 300 + rep)
        want = O.sort_u64(keys)
        for frac in (1.0, 0.6):
            n_del = int(n // k * frac)
            res = {}
            for flags in (0x4000, 0x0, 0x2000):
                heap = GeneralizedHeap(variant, k, n // k + 64, key_bits=32, debug_flags=flags, profile=True)
                heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
                heap.reset_counters()
                heap.profile(reset=True)
                d = heap.run_ops(phase_ops(1, n_del * k, k), np.zeros(0, np.uint32), n_del * k)
                out = d.out.reshape(-1, k)[np.argsort(d.seq, kind="stable")].reshape(-1).astype(np.uint64)
                c = heap.counters()
                p = heap.profile()
                rep_ = heap.check_invariants()
                resident = heap.collect_resident()
                res[flags] = (out, (c.merges, c.elided_merges, c.early_stops, c.propagation_node_visits, c.deletes),
                              rep_.ok, np.sort(resident), p["s3_ops"], p["del_served"])
                heap.close()
            ok = np.array_equal(res[0][0], want[: n_del * k]) and res[0][2]
            # (counters depend on the interleaving of concurrent heapifies;
            # outputs and the resident multiset do not)
            same = all(np.array_equal(res[0][0], res[f][0]) and np.array_equal(res[0][3], res[f][3])
                       for f in (0x4000, 0x2000))
            fails += not (ok and same)
            print(f"{variant.name} k={k} 2^{log2n} rep={rep} frac={frac}: sorted+inv={ok} same={same} "
                  f"counters s3={res[0x4000][1]} s2={res[0][1]} none={res[0x2000][1]} "
                  f"s3_ops={res[0x4000][4]} served={res[0x4000][5]}/{res[0][5]}", flush=True)
print(f"check_serve3: {fails} failures", flush=True)
