"""BASELINE configs 4 and 5 across GPUs (one process per GPU under torchrun):
SSSP sources and knapsack instances round-robin over ranks, one device heap
per rank, no data-path collective; the per-problem summaries are gathered
and rank 0 prints one JSON line per config with the max-over-ranks time.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/apps_multi.py [--sources 8] [--knapsack]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist

from paper_1906_06504_b200 import apps as A

ap = argparse.ArgumentParser()
ap.add_argument("--sources", type=int, default=8)
ap.add_argument("--knapsack", action="store_true")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl")
dm = dist if world > 1 else None
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))

g = A.grid_graph(2048, 2048, 1)
A.sssp(A.grid_graph(8, 8, 1), 0, device=local)  # context warm-up
cases = gold["grid_2048"][:a.sources]
if dm:
    dm.barrier()
t0 = time.perf_counter()
res = A.sssp_sources(g, [c["source"] for c in cases], device=local, dist_mod=dm)
t_local = time.perf_counter() - t0
t_max = t_local
if dm:
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    dm.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
exact = all({k: res[c["source"]][k] for k in ("sum", "max", "unreachable")} ==
            {k: c[k] for k in ("sum", "max", "unreachable")} for c in cases)
if rank == 0:
    print(json.dumps({"config": "sssp grid_graph(2048,2048,1), golden sources", "sources": len(cases),
                      "n_gpus": world, "seconds_max_over_ranks": round(t_max, 3), "exact": exact,
                      "per_source_s": {s: round(v["seconds"], 3) for s, v in sorted(res.items())}}), flush=True)
if a.knapsack:
    ref = json.load(open(os.path.join(ROOT, "tests", "golden", "knapsack_ref_bb_w1.json")))["cases"]
    solvable = [c for c in ref if "best" in c]
    insts = [A.generate_knapsack(A.KnapsackType(c["type"]), c["n"], c["range"], c["seed"]) for c in solvable]
    if dm:
        dm.barrier()
    t0 = time.perf_counter()
    kr = A.knapsack_instances(insts, device=local, dist_mod=dm)
    t_local = time.perf_counter() - t0
    t_max = t_local
    if dm:
        t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
        dm.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    exact = all(kr[i]["best"] == c["dp"] for i, c in enumerate(solvable))
    if rank == 0:
        print(json.dumps({"config": "knapsack golden instances the reference finishes", "instances": len(insts),
                          "n_gpus": world, "seconds_max_over_ranks": round(t_max, 3), "optimal": exact}), flush=True)
if dm:
    dm.barrier()
    dm.destroy_process_group()
