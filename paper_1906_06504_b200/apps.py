"""The heap's application drivers, mirroring the reference's interfaces.

* ``grid_graph`` / ``sssp``: ``proj/include/batchheap/{graph,sssp}.hpp``
  (``Graph``, ``SsspConfig``, ``SsspResult``, ``sssp``), implemented by
  ``bh_grid_graph`` / ``bh_sssp`` in the C ABI: BU device heap of 64-bit keys
  ``dist<<32 | node``, relaxation kernels, host loop over rounds
  (``proj/src/sssp.cpp:118-194``).
* ``generate_knapsack`` / ``knapsack_bb``:
  ``proj/include/batchheap/knapsack.hpp`` (``KnapsackType``,
  ``KnapsackInstance``, ``BbConfig``, ``BbOutcome``), implemented by
  ``bh_generate_knapsack`` / ``bh_knapsack_bb`` (``proj/src/knapsack.cpp``).

Multi-GPU: the heap does not shard, so independent
problems are spread over ranks -- SSSP sources and knapsack instances
round-robin, one heap per GPU, no collective on the data path; only the
per-problem summaries are gathered (``all_gather_object``) for reporting.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import _lib as L
from .heap import _raise

UNREACHABLE = (1 << 64) - 1  # kUnreachable (sssp.hpp:18-19)


@dataclasses.dataclass
class Graph:
    """CSR graph (proj/include/batchheap/graph.hpp:26-50): ``offsets`` (n+1),
    per-arc target ``nbr`` and ``weight``."""
    offsets: np.ndarray
    nbr: np.ndarray
    weight: np.ndarray

    @property
    def node_count(self) -> int:
        return int(self.offsets.size - 1)

    @property
    def edge_count(self) -> int:
        return int(self.nbr.size)


def grid_graph(rows: int, cols: int, seed: int) -> Graph:
    """grid_graph (proj/src/graph.cpp:174-193)."""
    lib = L.lib()
    m = int(lib.bh_grid_graph_edges(rows, cols))
    off = np.empty(rows * cols + 1, dtype=np.uint64)
    nbr = np.empty(max(m, 1), dtype=np.uint32)
    w = np.empty(max(m, 1), dtype=np.uint32)
    _raise(lib.bh_grid_graph(rows, cols, seed, off.ctypes.data_as(C.c_void_p),
                             nbr.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))
    return Graph(off, nbr[:m], w[:m])


@dataclasses.dataclass
class SsspConfig:
    """SsspConfig (sssp.hpp:27-31); ``ctas`` replaces the host worker count
    (0 = every co-resident CTA of the persistent heap kernel).  k defaults
    to 1024 (the reference: 32): device heap ops are latency-bound per op,
    so wide nodes are faster; the distances do not depend on k."""
    threshold: int = 10_000
    heap_node_capacity: int = 1024
    ctas: int = 0


@dataclasses.dataclass
class SsspResult:
    """SsspResult (sssp.hpp:21-24) plus run statistics."""
    dist: np.ndarray
    visits: int
    rounds: int = 0
    keys_through_heap: int = 0
    seconds: float = 0.0


def sssp(graph: Graph, source: int, config: Optional[SsspConfig] = None, device: int = 0) -> SsspResult:
    """sssp(graph, source, config) (proj/src/sssp.cpp:118-194) on the GPU."""
    cfg = config or SsspConfig()
    n = graph.node_count
    dist = np.empty(n, dtype=np.uint64)
    c = L.bh_sssp_cfg(cfg.threshold, cfg.heap_node_capacity, cfg.ctas, 0)
    st = L.bh_sssp_stats()
    off = np.ascontiguousarray(graph.offsets, dtype=np.uint64)
    nbr = np.ascontiguousarray(graph.nbr, dtype=np.uint32)
    w = np.ascontiguousarray(graph.weight, dtype=np.uint32)
    _raise(L.lib().bh_sssp(n, off.ctypes.data_as(C.c_void_p), nbr.ctypes.data_as(C.c_void_p),
                           w.ctypes.data_as(C.c_void_p), source, C.byref(c), device,
                           dist.ctypes.data_as(C.c_void_p), C.byref(st)))
    return SsspResult(dist, st.visits, st.rounds, st.keys_through_heap, st.seconds)


class KnapsackType(enum.IntEnum):
    """KnapsackType (knapsack.hpp:16-21)."""
    StronglyCorrelated = 0
    AlmostStronglyCorrelated = 1
    EvenOdd = 2
    SubsetSum = 3


TYPE_NAMES = {KnapsackType.StronglyCorrelated: "sc", KnapsackType.AlmostStronglyCorrelated: "asc",
              KnapsackType.EvenOdd: "esc", KnapsackType.SubsetSum: "ss"}  # knapsack_type_name


@dataclasses.dataclass
class KnapsackInstance:
    """KnapsackInstance (knapsack.hpp:23-31)."""
    type: KnapsackType
    n: int
    range: int
    weight: np.ndarray
    benefit: np.ndarray
    capacity: int


def generate_knapsack(kind: KnapsackType, n: int, rng_range: int, seed: int) -> KnapsackInstance:
    """generate_knapsack (proj/src/knapsack.cpp:22-66)."""
    w = np.empty(n, dtype=np.uint32)
    b = np.empty(n, dtype=np.uint32)
    cap = int(L.lib().bh_generate_knapsack(int(kind), n, rng_range, seed, w.ctypes.data_as(C.c_void_p),
                                           b.ctypes.data_as(C.c_void_p)))
    if cap == 0:
        _raise(L.BH_E_CONFIG)
    return KnapsackInstance(KnapsackType(kind), n, rng_range, w, b, cap)


@dataclasses.dataclass
class BbConfig:
    """BbConfig (knapsack.hpp:56-60): ``gc_threshold`` and
    ``heap_node_capacity`` as the reference; ``ctas`` replaces workers; a
    round pops ``pop_ops`` batches; ``arena_nodes`` node slots (recycled
    once a node is expanded or dropped) and ``max_explored`` (the node
    budget) bound a run.
    Defaults tuned on the device (tools/apps_sweep.py; the reference uses
    k = 32 and GC at 2^16 keys); the optimum does not depend on them."""
    gc_threshold: int = 1 << 20
    heap_node_capacity: int = 1024
    ctas: int = 0
    pop_ops: int = 4
    arena_nodes: int = 1 << 28
    max_explored: int = 1 << 29


@dataclasses.dataclass
class BbOutcome:
    """BbOutcome (knapsack.hpp:62-66) plus round statistics."""
    best: int
    explored: int
    gc_passes: int
    rounds: int = 0
    arena_nodes: int = 0
    seconds: float = 0.0


def knapsack_bb(instance: KnapsackInstance, config: Optional[BbConfig] = None, device: int = 0) -> BbOutcome:
    """knapsack_bb(instance, config) (proj/src/knapsack.cpp:206-368) on the
    GPU.  Raises CapacityError when the node slots or budget run out."""
    cfg = config or BbConfig()
    c = L.bh_bb_cfg(cfg.gc_threshold, cfg.heap_node_capacity, cfg.ctas, cfg.pop_ops, 0, cfg.arena_nodes,
                    cfg.max_explored)
    o = L.bh_bb_outcome()
    w = np.ascontiguousarray(instance.weight, dtype=np.uint32)
    b = np.ascontiguousarray(instance.benefit, dtype=np.uint32)
    _raise(L.lib().bh_knapsack_bb(instance.n, w.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                  instance.capacity, C.byref(c), device, C.byref(o)))
    return BbOutcome(o.best, o.explored, o.gc_passes, o.rounds, o.arena_nodes, o.seconds)


# ------------------------------------------------------------ multi-GPU --
def shard(items: Sequence, rank: int, world: int) -> List:
    """Round-robin share of `items` for `rank` (sources and
    instances are independent; no data-path collective)."""
    return [items[i] for i in range(rank, len(items), world)]


def dist_summary(dist: np.ndarray) -> dict:
    """Per-source fingerprint (the form of tests/golden/apps.json)."""
    reach = dist != np.uint64(UNREACHABLE)
    return {"sum": int(dist[reach].sum(dtype=np.uint64)), "max": int(dist[reach].max()) if reach.any() else 0,
            "unreachable": int((~reach).sum())}


def _gather(local: Dict, dist_mod) -> Dict:
    if dist_mod is None or not dist_mod.is_initialized() or dist_mod.get_world_size() == 1:
        return local
    parts: List[Optional[Dict]] = [None] * dist_mod.get_world_size()
    dist_mod.all_gather_object(parts, local)
    out: Dict = {}
    for p in parts:
        out.update(p)
    return out


def sssp_sources(graph: Graph, sources: Sequence[int], config: Optional[SsspConfig] = None,
                 solver: Optional[Callable[[Graph, int], np.ndarray]] = None, device: Optional[int] = None,
                 dist_mod=None) -> Dict[int, dict]:
    """Run `sources` round-robin over the ranks of `dist_mod`
    (torch.distributed, or None for one process), one device heap per rank;
    returns {source: summary} gathered on every rank.  `solver` defaults to
    the GPU driver (tests may pass a CPU oracle to exercise the sharding)."""
    rank = dist_mod.get_rank() if dist_mod is not None and dist_mod.is_initialized() else 0
    world = dist_mod.get_world_size() if dist_mod is not None and dist_mod.is_initialized() else 1
    dev = rank if device is None else device
    local: Dict[int, dict] = {}
    for s in shard(list(sources), rank, world):
        if solver is None:
            r = sssp(graph, s, config, device=dev)
            summ = dist_summary(r.dist)
            summ.update(visits=r.visits, rounds=r.rounds, seconds=r.seconds, rank=rank)
        else:
            summ = dist_summary(solver(graph, s))
            summ.update(rank=rank)
        local[int(s)] = summ
    return _gather(local, dist_mod)


def knapsack_instances(instances: Sequence[KnapsackInstance], config: Optional[BbConfig] = None,
                       solver: Optional[Callable[[KnapsackInstance], int]] = None, device: Optional[int] = None,
                       dist_mod=None) -> Dict[int, dict]:
    """Knapsack instances round-robin over ranks; {index: outcome} on every rank."""
    rank = dist_mod.get_rank() if dist_mod is not None and dist_mod.is_initialized() else 0
    world = dist_mod.get_world_size() if dist_mod is not None and dist_mod.is_initialized() else 1
    dev = rank if device is None else device
    local: Dict[int, dict] = {}
    for i in range(rank, len(instances), world):
        if solver is None:
            o = knapsack_bb(instances[i], config, device=dev)
            local[i] = {"best": o.best, "explored": o.explored, "gc_passes": o.gc_passes, "rounds": o.rounds,
                        "seconds": o.seconds, "rank": rank}
        else:
            local[i] = {"best": int(solver(instances[i])), "rank": rank}
    return _gather(local, dist_mod)
