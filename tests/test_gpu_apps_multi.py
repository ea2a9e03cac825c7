"""The multi-rank code path of the application drivers with the GPU solvers
(BASELINE configs 4 and 5; reference proj/src/sssp.cpp:118-194,
proj/src/knapsack.cpp:206-368): two ranks over gloo, each running its
round-robin share of SSSP sources and knapsack instances through the CUDA
drivers (bh_sssp / bh_knapsack_bb) -- both on cuda:0, the only GPU here --
then gathering the summaries.  Results are bit-exact against Dijkstra and
the DP optimum, each problem solved by the rank the round-robin assigns."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1906_06504_b200 import apps as A

pytestmark = pytest.mark.gpu

GRID = (96, 80, 5)
SOURCES = [0, 1234, 4000, 7679, 17, 3333]
KNAP = [(A.KnapsackType.StronglyCorrelated, 40, 1000, s) for s in (1, 2)] + \
       [(A.KnapsackType.SubsetSum, 50, 1000, s) for s in (1, 2, 3)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = A.grid_graph(*GRID)
        res = A.sssp_sources(g, SOURCES, A.SsspConfig(threshold=256), device=0, dist_mod=dist)
        insts = [A.generate_knapsack(*c) for c in KNAP]
        kn = A.knapsack_instances(insts, device=0, dist_mod=dist)
        q.put((rank, res, kn))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, repr(exc), None))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gpu_solvers_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, res, kn in got:
        assert kn is not None, res
    g = A.grid_graph(*GRID)
    exp_sssp = {s: A.dist_summary(O.dijkstra(g.offsets, g.nbr, g.weight, s)) for s in SOURCES}
    insts = [A.generate_knapsack(*c) for c in KNAP]
    exp_kn = [O.knapsack_dp(i.weight, i.benefit, i.capacity) for i in insts]
    for rank, res, kn in got:
        assert sorted(res) == sorted(SOURCES)
        for i, s in enumerate(SOURCES):
            assert {k: res[s][k] for k in exp_sssp[s]} == exp_sssp[s], (rank, s)
            assert res[s]["rank"] == i % world
            assert res[s]["visits"] > 0  # solved on the device heap
        assert sorted(kn) == list(range(len(KNAP)))
        for i in range(len(KNAP)):
            assert kn[i]["best"] == exp_kn[i], (rank, i)
            assert kn[i]["rank"] == i % world
            assert kn[i]["explored"] > 0
