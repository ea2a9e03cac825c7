"""Application drivers, host side (no GPU): the product library's instance
generators against the oracle and the reference's golden fixtures, and the
multi-rank sharding of independent problems (gloo, world size 2)."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1906_06504_b200 import apps as A

ROOT = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(ROOT, "golden", "apps.json")))


@pytest.mark.parametrize("rows,cols,seed", [(64, 64, 1), (3, 7, 5), (1, 9, 2), (128, 96, 11)])
def test_grid_graph_matches_oracle(rows, cols, seed):
    g = A.grid_graph(rows, cols, seed)
    off, nbr, w = O.grid_graph(rows, cols, seed)
    assert np.array_equal(g.offsets, off)
    assert np.array_equal(g.nbr, nbr) and np.array_equal(g.weight, w)
    assert g.edge_count == 2 * (rows * (cols - 1) + (rows - 1) * cols)


def test_grid_graph_small_golden_distances():
    """The reference's Dijkstra on its own grid_graph(64, 64, 1) (golden),
    reproduced by the oracle on the product's graph."""
    case = GOLD["grid_small"][0]
    g = A.grid_graph(case["rows"], case["cols"], case["seed"])
    d = O.dijkstra(g.offsets, g.nbr, g.weight, case["source"])
    assert d.tolist() == case["dist"]


def test_knapsack_generator_matches_golden():
    for case in GOLD["knapsack"]:
        inst = A.generate_knapsack(A.KnapsackType(case["type"]), case["n"], case["range"], case["seed"])
        assert inst.capacity == case["capacity"]
        assert inst.weight[:4].tolist() == case["w_head"] and inst.benefit[:4].tolist() == case["b_head"]
        w, b, cap = O.generate_knapsack(case["type"], case["n"], case["range"], case["seed"])
        assert np.array_equal(inst.weight, w) and np.array_equal(inst.benefit, b) and cap == inst.capacity


def test_knapsack_generator_rejects_bad_args():
    with pytest.raises(RuntimeError):
        A.generate_knapsack(A.KnapsackType.SubsetSum, 0, 1000, 1)


def test_shard_round_robin():
    items = list(range(8))
    for world in (1, 2, 4, 8):
        parts = [A.shard(items, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == items
        assert all(len(p) == 8 // world for p in parts)


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
        g = A.grid_graph(24, 24, 3)
        sources = [0, 100, 200, 300, 400, 500, 575, 17]
        res = A.sssp_sources(g, sources, solver=lambda gr, s: O.dijkstra(gr.offsets, gr.nbr, gr.weight, s),
                             dist_mod=dist)
        insts = [A.generate_knapsack(A.KnapsackType(t), 30, 1000, s) for t in (0, 3) for s in (1, 2, 3)]
        kn = A.knapsack_instances(insts, solver=lambda i: O.knapsack_dp(i.weight, i.benefit, i.capacity),
                                  dist_mod=dist)
        q.put((rank, res, kn))
    finally:
        dist.destroy_process_group()


def test_multi_rank_sharding_gloo():
    """world_size 2 over gloo on CPU: every source / instance is solved by
    exactly the rank the round-robin assigns, and every rank ends with the
    full set of results, equal to a single-process run."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = A.grid_graph(24, 24, 3)
    sources = [0, 100, 200, 300, 400, 500, 575, 17]
    for rank, res, kn in got:
        assert sorted(res) == sorted(sources)
        for i, s in enumerate(sources):
            exp = A.dist_summary(O.dijkstra(g.offsets, g.nbr, g.weight, s))
            assert {k: res[s][k] for k in exp} == exp
            assert res[s]["rank"] == i % world
        assert sorted(kn) == list(range(6))
        for i in range(6):
            assert kn[i]["rank"] == i % world
    insts = [A.generate_knapsack(A.KnapsackType(t), 30, 1000, s) for t in (0, 3) for s in (1, 2, 3)]
    for i, inst in enumerate(insts):
        assert got[0][2][i]["best"] == O.knapsack_dp(inst.weight, inst.benefit, inst.capacity)
