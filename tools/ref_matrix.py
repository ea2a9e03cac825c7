"""CPU baseline matrix: the
reference's own GeneralizedHeap (oracle/_ref, compiled from
/root/reference/proj/src) on this host: TD and BU, each with 1 worker and
with every host thread, phase-split timer (insert-all then deleteMin-all),
plus the reference's run_workload rows (proj/src/workload.cpp:75-147,
proj/src/bench.cpp:60-113): insert-all-then-delete-all and config 3's
ins-del pairs on 14 seeded levels.  Writes JSON (tooling; run on the GPU box:
python tools/ref_matrix.py profiles/r2/ref_matrix.json)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle as O

out_path = sys.argv[1] if len(sys.argv) > 1 else "ref_matrix.json"
nproc = len(os.sched_getaffinity(0))
k = 1024
rows = []
for variant, vname in ((0, "td"), (1, "bu")):
    for workers in (1, nproc):
        log2n = 24 if workers == 1 else 26
        n = 1 << log2n
        ti, td = O.ref_phase(variant, k, n, workers, 1, False)
        rows.append({"kind": "phase", "variant": vname, "workers": workers, "log2n": log2n, "k": k,
                     "insert_s": ti, "delete_s": td, "key_ops_per_s": 2 * n / (ti + td)})
        print(json.dumps(rows[-1]), flush=True)
r = O.ref()
for variant, vname in ((1, "bu"), (0, "td")):
    for pattern, pname, full in ((1, "ins_del_pairs", 100), (0, "insert_all_then_delete_all", 100)):
        out = np.zeros(7, np.float64)
        st = r.ref_run_workload(variant, k, nproc, 1 << 26, 0, pattern, 14 if pattern == 1 else 0, full, 1, out)
        rows.append({"kind": "run_workload", "variant": vname, "pattern": pname, "full_batch_pct": full,
                     "workers": nproc, "initial_levels": 14 if pattern == 1 else 0, "total_keys": 1 << 26, "k": k, "status": st,
                     "wall_s": out[0], "ops": out[1], "key_ops_per_s": 2 * (1 << 26) / out[0] if out[0] else None})
        print(json.dumps(rows[-1]), flush=True)
os.makedirs(os.path.dirname(os.path.abspath(out_path)), exist_ok=True)
with open(out_path, "w") as f:
    json.dump({"host_threads": nproc, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
               if os.path.exists("/proc/cpuinfo") else None,
               "generated": time.strftime("%Y-%m-%d %H:%M:%S"), "rows": rows}, f, indent=1)
