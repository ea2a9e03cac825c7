import sys, os
sys.path.insert(0, "/root/repo")
from oracle import oracle as O
from paper_1906_06504_b200 import apps as A
inst = A.generate_knapsack(A.KnapsackType(0), 100, 1000, 1)
print("dp", O.knapsack_dp(inst.weight, inst.benefit, inst.capacity))
for cfg in (A.BbConfig(), A.BbConfig(arena_nodes=1 << 28), A.BbConfig(heap_node_capacity=256, pop_ops=4), A.BbConfig(heap_node_capacity=32, pop_ops=16, gc_threshold=1<<16)):
    try:
        o = A.knapsack_bb(inst, cfg)
        print(cfg, o)
    except Exception as e:
        print(cfg, type(e).__name__, e)
