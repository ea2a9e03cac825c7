"""Quick GPU probe of the application drivers: exactness + timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle as O
from paper_1906_06504_b200 import apps as A

for rows, k, thr in ((64, 32, 200), (256, 32, 10000), (256, 1024, 10000), (512, 32, 10000), (512, 1024, 10000)):
    g = A.grid_graph(rows, rows, 1)
    t = time.time()
    r = A.sssp(g, 0, A.SsspConfig(threshold=thr, heap_node_capacity=k))
    exp = O.dijkstra(g.offsets, g.nbr, g.weight, 0)
    print(f"sssp {rows}x{rows} k={k} thr={thr}: exact={np.array_equal(r.dist, exp)} {r.seconds:.3f}s "
          f"rounds={r.rounds} visits={r.visits} heap_keys={r.keys_through_heap}", flush=True)
for t_, n, R, s in ((0, 50, 1000, 1), (3, 50, 1000, 1), (0, 200, 1000, 1), (0, 200, 7000, 1), (3, 200, 7000, 1),
                    (1, 50, 1000, 1), (2, 50, 1000, 1)):
    inst = A.generate_knapsack(A.KnapsackType(t_), n, R, s)
    dp = O.knapsack_dp(inst.weight, inst.benefit, inst.capacity)
    try:
        o = A.knapsack_bb(inst)
        print(f"knapsack {A.TYPE_NAMES[A.KnapsackType(t_)]} n={n} R={R} s={s}: best={o.best} dp={dp} "
              f"exact={o.best == dp} {o.seconds:.3f}s explored={o.explored} rounds={o.rounds} gc={o.gc_passes}",
              flush=True)
    except Exception as e:
        print(f"knapsack {t_} n={n} R={R}: {type(e).__name__}: {e}", flush=True)
