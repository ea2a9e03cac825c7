"""The reference's knapsack_bb (oracle/_ref, unmodified sources) on every
golden knapsack instance, one child process each (arena exhaustion calls
std::terminate in the reference).  Writes tests/golden/knapsack_ref_bb.json:
per instance the optimum/explored/seconds, or the failure.
usage: ref_knapsack_table.py [WORKERS] [TIMEOUT_S] [OUT_JSON]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))["knapsack"]
workers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
timeout = float(sys.argv[2]) if len(sys.argv) > 2 else 30
out = []
for c in gold:
    r = O.ref_knapsack_bb_subprocess(c["type"], c["n"], c["range"], c["seed"], workers=workers, timeout=timeout)
    r.update({k: c[k] for k in ("type", "n", "range", "seed", "dp")})
    r["workers"] = workers
    out.append(r)
    print(r, flush=True)
path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "tests", "golden", f"knapsack_ref_bb_w{workers}.json")
json.dump({"generator": "tools/ref_knapsack_table.py", "timeout_s": timeout, "cases": out}, open(path, "w"), indent=0)
