"""Application drivers on the GPU (BASELINE configs 4 and 5): SSSP distances
bit-exact against Dijkstra (the oracle and the reference's golden fixtures),
knapsack branch-and-bound optimum equal to the DP oracle."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1906_06504_b200 import apps as A

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(ROOT, "golden", "apps.json")))


def test_sssp_grid_small_golden():
    case = GOLD["grid_small"][0]
    g = A.grid_graph(case["rows"], case["cols"], case["seed"])
    r = A.sssp(g, case["source"], A.SsspConfig(threshold=200))
    assert r.dist.tolist() == case["dist"]
    assert r.keys_through_heap > 0  # the heap was engaged


@pytest.mark.parametrize("k", [32, 1024])
@pytest.mark.parametrize("threshold", [64, 10_000])
def test_sssp_matches_dijkstra(k, threshold):
    g = A.grid_graph(192, 160, 7)
    for s in (0, 12345, g.node_count - 1):
        r = A.sssp(g, s, A.SsspConfig(threshold=threshold, heap_node_capacity=k))
        exp = O.dijkstra(g.offsets, g.nbr, g.weight, s)
        assert np.array_equal(r.dist, exp), (k, threshold, s)


def test_sssp_disconnected_and_errors():
    # a unit-width grid is a path graph
    g = A.grid_graph(1, 50, 3)
    r = A.sssp(g, 10, A.SsspConfig(threshold=8))
    assert np.array_equal(r.dist, O.dijkstra(g.offsets, g.nbr, g.weight, 10))
    from paper_1906_06504_b200 import ConfigError
    with pytest.raises(ConfigError):
        A.sssp(g, 50)


@pytest.mark.slow
def test_sssp_grid_2048_golden_source0():
    g = A.grid_graph(2048, 2048, 1)
    case = GOLD["grid_2048"][0]
    r = A.sssp(g, case["source"], A.SsspConfig(heap_node_capacity=1024))
    assert A.dist_summary(r.dist) == {k: case[k] for k in ("sum", "max", "unreachable")}


# Golden instances (all four families) whose branch-and-bound exceeds the
# default node budget (2^29 nodes) on the GPU too -- the reference
# terminates on a superset of these, tests/golden/knapsack_ref_bb_w1.json --
# and the ones that take seconds.
EXHAUST = {(0, 100, 1000, 3), (0, 200, 1000, 2), (0, 200, 7000, 2), (1, 200, 1000, 1), (1, 200, 7000, 1),
           (2, 200, 1000, 1), (2, 200, 1000, 3), (2, 200, 7000, 1)}
SLOW = {(0, 100, 1000, 1), (0, 100, 7000, 1), (1, 100, 1000, 1), (1, 100, 7000, 1), (1, 200, 7000, 2),
        (2, 200, 7000, 2)}


def _key(c):
    return (c["type"], c["n"], c["range"], c["seed"])


def _cases():
    for c in GOLD["knapsack"]:
        if _key(c) in EXHAUST:
            continue
        marks = [pytest.mark.slow] if _key(c) in SLOW else []
        yield pytest.param(c, marks=marks, id="t%d-n%d-R%d-s%d" % _key(c))


@pytest.mark.parametrize("case", list(_cases()))
def test_knapsack_bb_matches_dp_golden(case):
    inst = A.generate_knapsack(A.KnapsackType(case["type"]), case["n"], case["range"], case["seed"])
    out = A.knapsack_bb(inst)
    assert out.best == case["dp"]
    assert out.explored > 0


def test_knapsack_bb_solves_what_the_reference_solves():
    """Every golden instance the reference's B&B finishes (W=1,
    tests/golden/knapsack_ref_bb_w1.json) is outside EXHAUST."""
    ref = json.load(open(os.path.join(ROOT, "golden", "knapsack_ref_bb_w1.json")))["cases"]
    solved = {_key(c) for c in ref if "best" in c}
    assert solved and not (solved & EXHAUST)
    assert all(c["best"] == c["dp"] for c in ref if "best" in c)


def test_knapsack_bb_arena_exhaustion_raises():
    """The reference's "branch-and-bound arena exhausted" (knapsack.cpp:
    136-154) is a CapacityError here instead of std::terminate."""
    from paper_1906_06504_b200 import CapacityError
    inst = A.generate_knapsack(A.KnapsackType.StronglyCorrelated, 200, 1000, 2)
    with pytest.raises(CapacityError, match="budget"):
        A.knapsack_bb(inst, A.BbConfig(max_explored=1 << 20))
    with pytest.raises(CapacityError, match="arena"):
        A.knapsack_bb(inst, A.BbConfig(arena_nodes=1 << 12))


@pytest.mark.parametrize("k,pop", [(32, 1), (32, 64), (256, 16)])
def test_knapsack_bb_shapes(k, pop):
    for t in (A.KnapsackType.StronglyCorrelated, A.KnapsackType.SubsetSum):
        inst = A.generate_knapsack(t, 60, 1000, 9)
        out = A.knapsack_bb(inst, A.BbConfig(heap_node_capacity=k, pop_ops=pop, gc_threshold=1 << 12))
        assert out.best == O.knapsack_dp(inst.weight, inst.benefit, inst.capacity)


def test_knapsack_bb_small_asc_esc():
    for t in (A.KnapsackType.AlmostStronglyCorrelated, A.KnapsackType.EvenOdd):
        inst = A.generate_knapsack(t, 40, 1000, 4)
        out = A.knapsack_bb(inst)
        assert out.best == O.knapsack_dp(inst.weight, inst.benefit, inst.capacity)
