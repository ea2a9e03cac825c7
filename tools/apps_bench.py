"""BASELINE configs 4 and 5 on one GPU, next to the reference's CPU drivers.

* SSSP: grid_graph(2048, 2048, 1), the 8 sources i*524288; GPU driver
  (device defaults) -> per-source seconds and exactness vs the reference's
  golden distance fingerprints (tests/golden/apps.json); the reference's
  sssp() (oracle/_ref, unmodified sources, workers = host cores) timed on
  the first source.
* Knapsack: the golden sc / ss / asc / esc instances the reference's B&B
  finishes (tests/golden/knapsack_ref_bb_w1.json), GPU time vs the
  reference's recorded time; optimum vs knapsack_dp.
Multi-GPU: the same problems spread round-robin over ranks (apps.sssp_sources
/ apps.knapsack_instances) -- replicas, no collective."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_1906_06504_b200 import apps as A

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))
n_src = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t0 = time.time()
g = A.grid_graph(2048, 2048, 1)
print(f"grid_graph 2048^2: {g.node_count} nodes {g.edge_count} arcs ({time.time() - t0:.1f}s host)", flush=True)
A.sssp(A.grid_graph(8, 8, 1), 0)  # context warm-up
tot = 0.0
for case in gold["grid_2048"][:n_src]:
    r = A.sssp(g, case["source"])
    ok = A.dist_summary(r.dist) == {k: case[k] for k in ("sum", "max", "unreachable")}
    tot += r.seconds
    print(f"sssp source {case['source']:8d}: {r.seconds:.3f}s exact={ok} rounds={r.rounds} visits={r.visits} "
          f"heap_keys={r.keys_through_heap}", flush=True)
print(f"sssp {n_src} sources on 1 GPU: {tot:.2f}s", flush=True)
try:
    import ctypes as C
    from oracle import oracle as O
    d = np.empty(g.node_count, np.uint64)
    v, s = C.c_uint64(), C.c_double()
    w = os.cpu_count()
    st = O.ref().ref_grid_sssp(2048, 2048, 1, 0, 10000, w, d, C.byref(v), C.byref(s))
    print(f"reference sssp (CPU, {w} workers) source 0: {s.value:.3f}s status={st} "
          f"exact={A.dist_summary(d) == {k: gold['grid_2048'][0][k] for k in ('sum', 'max', 'unreachable')}}",
          flush=True)
except Exception as e:
    print("reference sssp unavailable:", e)
ref = json.load(open(os.path.join(ROOT, "tests", "golden", "knapsack_ref_bb_w1.json")))["cases"]
gt = rt = 0.0
n = 0
for c in ref:
    if "best" not in c:
        continue
    inst = A.generate_knapsack(A.KnapsackType(c["type"]), c["n"], c["range"], c["seed"])
    o = A.knapsack_bb(inst)
    assert o.best == c["dp"], c
    gt += o.seconds
    rt += c["seconds"]
    n += 1
print(f"knapsack: {n} instances the reference finishes, all optimal on the GPU; GPU {gt:.2f}s total vs "
      f"reference B&B (1 worker, survey container) {rt:.2f}s", flush=True)
