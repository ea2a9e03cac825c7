"""All golden knapsack instances on the GPU driver: optimum vs DP, time."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_06504_b200 import apps as A

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))["knapsack"]
only = {tuple(map(int, a.split(","))) for a in sys.argv[1:]}
if only:
    gold = [c for c in gold if (c["type"], c["n"], c["range"], c["seed"]) in only]
A.sssp(A.grid_graph(8, 8, 1), 0)
res = []
for c in gold:
    inst = A.generate_knapsack(A.KnapsackType(c["type"]), c["n"], c["range"], c["seed"])
    try:
        o = A.knapsack_bb(inst)
        r = {"best": o.best, "ok": o.best == c["dp"], "seconds": round(o.seconds, 3), "explored": o.explored}
    except Exception as e:
        r = {"error": f"{type(e).__name__}: {e}"}
    r.update({k: c[k] for k in ("type", "n", "range", "seed", "dp")})
    res.append(r)
    print(r, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "kn_golden_gpu.json"), "w"), indent=0)
