"""Round-shape sweep for the knapsack B&B and SSSP drivers (timings only;
exactness checked against the oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_1906_06504_b200 import apps as A

A.sssp(A.grid_graph(16, 16, 1), 0)  # warm the context
for t_, n, R in ((0, 200, 1000), (0, 200, 7000), (3, 200, 7000)):
    inst = A.generate_knapsack(A.KnapsackType(t_), n, R, 1)
    dp = O.knapsack_dp(inst.weight, inst.benefit, inst.capacity)
    for k in (32, 256, 1024):
        for pop in (1, 4, 16):
            for gc in (1 << 16, 1 << 20):
                o = A.knapsack_bb(inst, A.BbConfig(heap_node_capacity=k, pop_ops=pop, gc_threshold=gc))
                print(f"{A.TYPE_NAMES[A.KnapsackType(t_)]} n={n} R={R} k={k} pop={pop} gc={gc}: ok={o.best == dp} "
                      f"{o.seconds:.3f}s explored={o.explored} rounds={o.rounds} gcs={o.gc_passes}", flush=True)
g = A.grid_graph(1024, 1024, 1)
for k in (32, 256, 1024, 2048):
    for thr in (10000, 50000):
        r = A.sssp(g, 0, A.SsspConfig(threshold=thr, heap_node_capacity=k))
        print(f"sssp 1024^2 k={k} thr={thr}: {r.seconds:.3f}s rounds={r.rounds} visits={r.visits}", flush=True)
