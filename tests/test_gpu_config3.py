"""BASELINE config 3 on the kernel that is timed (GPU).

* Recorded histories at K=1024 from the production schedule: the recorded
  kernel runs the same lock schedule as the unrecorded one (the refill of the
  last node beside the claim of the root's / the server's children, marked as
  refill spans in the log), with all co-resident CTAs, a heap seeded with 255
  nodes so delete serving engages, then >= 4096 coin-flip 50/50 ops with 20%
  partial inserts (proj/src/workload.cpp:99-120).  The history
  goes through the reference's checkers: check_td / check_bu (constructive
  orders, proj/src/lincheck.cpp:53-86), the just-in-time witness builder,
  mutual exclusion and lock order (lincheck.cpp:156-217), and the BU overlap
  windows (lincheck.cpp:219-241).
* Full size, unrecorded: 14 seeded levels (16383 nodes of generate_keys with
  the reference's seed, proj/src/bench.cpp:60-72), then 2^26 keys of insert
  traffic, as strict ins-del pairs (bench.cpp:105-113) and as coin-flip 50/50
  with 20% partial inserts.  Multiset conservation (deleted + resident ==
  seed + inserted, workload.cpp:135-145) and the quiescent invariants
  (heap.cpp:726-770).
"""
import numpy as np
import pytest

from oracle import lincheck as LC
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, make_ops, phase_ops

pytestmark = pytest.mark.gpu

K = 1024
SEED_LEVELS_SMALL = 8  # 255 nodes: above the 64 a delete server needs


def coin_flip_ops(rng, n_ops, k, partial_pct, key_hi, seed_nodes=0, dtype=np.uint64, tail_deletes=0):
    """Seed inserts (full batches) first, then coin-flip 50/50 ins/del with
    partial_pct % of the inserts partial (1..k-1 keys), then tail_deletes
    deletes in a row."""
    kinds, lens, offs, chunks = [], [], [], []
    at = out_at = 0
    for _ in range(seed_nodes):
        chunks.append(rng.integers(0, key_hi, size=k, dtype=np.uint64))
        kinds.append(0); lens.append(k); offs.append(at)
        at += k
    for _ in range(n_ops):
        if rng.integers(0, 2) == 0:
            n = k if rng.integers(0, 100) >= partial_pct else int(rng.integers(1, k))
            chunks.append(rng.integers(0, key_hi, size=n, dtype=np.uint64))
            kinds.append(0); lens.append(n); offs.append(at)
            at += n
        else:
            kinds.append(1); lens.append(0); offs.append(out_at)
            out_at += k
    for _ in range(tail_deletes):
        kinds.append(1); lens.append(0); offs.append(out_at)
        out_at += k
    ops = make_ops(np.array(kinds, np.uint32), np.array(lens, np.uint32), np.array(offs, np.uint64))
    return ops, np.concatenate(chunks).astype(dtype), out_at


def recorded_history(heap, ops, r, pool):
    ev = heap.history_events()
    keys = []
    for i, o in enumerate(ops):
        if o["kind"] == 0:
            keys.append(pool[o["offset"]:o["offset"] + o["len"]].tolist())
        else:
            keys.append(r.out[o["offset"]:o["offset"] + r.lens[i]].tolist())
    skip = {i for i in range(len(ops)) if r.status[i] not in (0, 3)}
    return LC.decode_history(ev, ops["kind"], keys, skip)


def refill_overlaps(hist):
    """Refill spans still held when the same op claimed one of the refill
    node's ancestors: the production split schedule, visible in the log."""
    n = 0
    for op in hist:
        for a in op.locks:
            if not a.refill:
                continue
            for b in op.locks:
                if b is a or b.node == a.node:
                    continue
                if a.acquire_ts < b.acquire_ts < a.release_ts and LC._is_ancestor(b.node, a.node):
                    n += 1
    return n


@pytest.mark.slow
@pytest.mark.parametrize("partial_pct", [20, 0])
@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
def test_recorded_k1024_coin_flip_linearizable(variant, partial_pct):
    """partial_pct=20: the reference's mix.  partial_pct=0: full batches
    only, so the partial buffer stays empty and the burst of deletes at the
    end is served (delete serving needs an empty partial buffer; the coin-flip
    phase rarely queues two deletes back to back, BU deletes waiting outside
    the root queue while climbs run)."""
    rng = np.random.default_rng(20261017 + int(variant) + partial_pct)
    seed_nodes = (1 << SEED_LEVELS_SMALL) - 1
    ops, pool, out_len = coin_flip_ops(rng, 4096, K, partial_pct, (1 << 32) - 1, seed_nodes, np.uint32,
                                       tail_deletes=128)
    heap = GeneralizedHeap(variant, K, seed_nodes + len(ops) + 8, key_bits=32, record=True, profile=True)
    r = heap.run_ops(ops, pool, out_len)  # ctas=0: every co-resident CTA
    assert heap.info()["max_ctas"] >= 100
    assert set(np.unique(r.status).tolist()) <= {0, 3}
    p = heap.profile()
    hist = recorded_history(heap, ops, r, pool)
    assert len(hist) == len(ops)
    assert LC.validate(hist) is None
    ok, why = LC.check_mutual_exclusion(hist)
    assert ok, why
    ok, why = LC.check_lock_order(hist)
    assert ok, why
    res = LC.check_td(hist, K) if variant == Variant.TD else LC.check_bu(hist, K)
    assert res.passed, res.detail
    jit = LC.check_jit(hist, K)
    assert jit.passed, jit.detail
    if variant == Variant.BU:
        ok, why = LC.check_bu_overlap_windows(hist)
        assert ok, why
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    # the history covers the timed kernel's schedule: refills overlapping
    # the claim of an ancestor, and (full batches) served deletes
    assert refill_overlaps(hist) > 0
    if partial_pct == 0:
        assert p["del_served"] > 0
    deleted = np.concatenate([r.out[o["offset"]:o["offset"] + r.lens[i]]
                              for i, o in enumerate(ops) if o["kind"] == 1])
    acc = np.sort(np.concatenate([deleted.astype(np.uint64), heap.collect_resident()]))
    assert np.array_equal(acc, np.sort(pool.astype(np.uint64)))


def _seed_heap(variant, extra_nodes):
    levels = 14
    seed_nodes = (1 << levels) - 1
    seed_keys = O.generate_keys(seed_nodes * K, 1 ^ 0x5851F42D4C957F2D).astype(np.uint32)
    heap = GeneralizedHeap(variant, K, seed_nodes + extra_nodes + 256, key_bits=32)
    r = heap.run_ops(phase_ops(0, seed_keys.size, K), seed_keys, 0)
    assert np.all(r.status == 0)
    return heap, seed_keys


def _check_conservation(heap, r, ops, seed_keys, pool):
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    dmask = ops["kind"] == 1
    lens = r.lens[dmask]
    offs = ops["offset"][dmask].astype(np.int64)
    full = lens == K
    if full.all():
        deleted = r.out.reshape(-1, K)[(offs // K)].reshape(-1) if offs.size else np.zeros(0, np.uint32)
    else:
        deleted = np.concatenate([r.out[o:o + n] for o, n in zip(offs, lens)])
    left = np.sort(np.concatenate([deleted.astype(np.uint32), heap.collect_resident().astype(np.uint32)]))
    right = np.sort(np.concatenate([seed_keys, pool]))
    assert left.size == right.size
    assert np.array_equal(left, right)


@pytest.mark.slow
def test_config3_full_size_strict_pairs_bu():
    """14 seeded levels, 2^16 ins-del pairs of full K=1024 batches (2^26 keys
    of inserts), BU."""
    pairs = 1 << 16
    heap, seed_keys = _seed_heap(Variant.BU, pairs)
    rng = np.random.default_rng(7)
    pool = rng.integers(0, (1 << 32) - 1, size=pairs * K, dtype=np.uint64).astype(np.uint32)
    kinds = np.tile(np.array([0, 1], np.uint32), pairs)
    lens = np.tile(np.array([K, 0], np.uint32), pairs)
    offs = np.repeat(np.arange(pairs, dtype=np.uint64) * np.uint64(K), 2)
    ops = make_ops(kinds, lens, offs)
    r = heap.run_ops(ops, pool, pairs * K)
    assert np.all(r.status == 0)
    _check_conservation(heap, r, ops, seed_keys, pool)


@pytest.mark.slow
@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
def test_config3_full_size_coin_flip_partials(variant):
    """14 seeded levels, then coin-flip 50/50 ins/del with 20% partial
    inserts until 2^26 keys have been inserted."""
    rng = np.random.default_rng(11 + int(variant))
    n_ops = int((1 << 26) / (0.5 * (0.8 * K + 0.2 * K / 2)))
    ops, pool, out_len = coin_flip_ops(rng, n_ops, K, 20, (1 << 32) - 1, 0, np.uint32)
    heap, seed_keys = _seed_heap(variant, n_ops)
    r = heap.run_ops(ops, pool, out_len)
    assert set(np.unique(r.status).tolist()) <= {0}
    assert pool.size >= (1 << 26) * 0.95
    _check_conservation(heap, r, ops, seed_keys, pool)
