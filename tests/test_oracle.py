"""CPU suite: the oracle pinned against the reference's golden vectors and
known-answer tests, before it is trusted as the
checker of the CUDA path."""
import json
import os

import numpy as np
import pytest
from sortedcontainers import SortedList

from oracle import lincheck as LC
from oracle import oracle as O

ROOT = os.path.dirname(os.path.abspath(__file__))


def golden(name):
    with open(os.path.join(ROOT, "golden", name)) as f:
        return json.load(f)


# ------------------------------------------------------------- keygen ----
def test_keygen_2pow20_matches_reference_golden():
    g = golden("keygen.json")["20"]
    keys = O.generate_keys(g["n"], g["seed"])
    assert keys[:8].tolist() == g["first"]
    s = O.sort_u64(keys)
    assert (int(s[0]), int(s[-1])) == (g["min"], g["max"])
    assert O.checksums(s) == (g["sum"], g["xor"], g["poly_hash"])
    assert int((s[1:] == s[:-1]).sum()) == g["adjacent_dups"]
    # SURVEY Appendix B, quoted values
    assert keys[:3].tolist() == [574995807, 585863760, 1937953255]
    assert g["sum"] == 2251638043183164 and g["xor"] == 1757954550


def test_keygen_orders():
    g = golden("keygen.json")
    assert O.generate_keys(16, 3, O.ASCEND).tolist() == g["order1"]
    assert O.generate_keys(16, 3, O.DESCEND).tolist() == g["order2"]


def test_keygen_2pow26_prefix_and_no_u32_sentinel():
    g = golden("keygen.json")["26"]
    keys = O.generate_keys(1 << 22, 1)
    assert keys[:8].tolist() == g["first"]
    assert g["count_u32_sentinel"] == 0


# ------------------------------------------------------- batch KATs ------
def test_merge_kats():
    hi, lo = O.merge_and_sort([1, 3, 5, 7], [2, 4, 6, 8], 4)
    assert hi.tolist() == [1, 2, 3, 4] and lo.tolist() == [5, 6, 7, 8]
    hi, lo = O.merge_and_sort([1, 2], [], 4)
    assert hi.tolist() == [1, 2] and lo.size == 0
    hi, lo = O.merge_and_sort([5, 5], [5], 2)
    assert hi.tolist() == [5, 5] and lo.tolist() == [5]


def test_merge_equals_concat_sort_split():
    rng = np.random.default_rng(7)
    for _ in range(500):
        k = 1 << int(rng.integers(0, 6))
        a = np.sort(rng.integers(0, 1001, size=int(rng.integers(0, 2 * k))).astype(np.uint64))
        b = np.sort(rng.integers(0, 1001, size=int(rng.integers(0, 2 * k)) + 1).astype(np.uint64))
        hi, lo = O.merge_and_sort(a, b, k)
        c = np.sort(np.concatenate([a, b]))
        cut = min(k, c.size)
        assert hi.tolist() == c[:cut].tolist() and lo.tolist() == c[cut:].tolist()


def test_needs_merge_kats():
    assert not O.needs_merge([1, 2], [3, 4])
    assert O.needs_merge([1, 4], [2, 3])
    assert not O.needs_merge([5, 6], [1, 2])


def test_needs_merge_soundness():
    rng = np.random.default_rng(11)
    elided = 0
    for _ in range(2000):
        a = np.sort(rng.integers(0, 41, size=4).astype(np.uint64))
        b = np.sort(rng.integers(0, 41, size=4).astype(np.uint64))
        if O.needs_merge(a, b):
            continue
        elided += 1
        hi, lo = O.merge_and_sort(a, b, 4)
        assert (hi.tolist() == a.tolist() and lo.tolist() == b.tolist()) or \
               (hi.tolist() == b.tolist() and lo.tolist() == a.tolist())
    assert elided > 0


# ------------------------------------------------------------ bitrev ----
def test_bit_reverse_kat():
    assert [O.bit_reverse(c, 3) for c in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]
    assert O.bit_reverse(0, 0) == 0 and O.slot_for_rank(1) == 1


def test_slot_for_rank_bijection_and_paths():
    for level in range(8):
        base = 1 << level
        slots = {O.slot_for_rank(r) for r in range(base, 2 * base)}
        assert slots == set(range(base, 2 * base))
    for level in range(1, 7):
        base = 1 << level
        for r in range(base, 2 * base - 1):
            p1 = set(O.path_to_slot(O.slot_for_rank(r)))
            p2 = O.path_to_slot(O.slot_for_rank(r + 1))
            assert sum(n in p1 for n in p2) == 1


# --------------------------------------------------------- seq heap ------
def test_seqheap_replays_reference_histories_exactly():
    """The oracle's sequential heap returns the reference GeneralizedHeap's
    results and counters op for op on every golden history."""
    for case in golden("heap_histories.json"):
        h = O.SeqHeap(case["variant"], case["k"], case["max_nodes"], case["elide"])
        for kind, arg, res, st in zip(case["ops"], case["args"], case["results"], case["statuses"]):
            if kind == 0:
                assert h.insert(np.array(arg, dtype=np.uint64)) == st
            else:
                got_st, got = h.delete_min()
                assert got_st == st
                assert got.tolist() == res
        assert h.counters() == case["counters"]


def test_seqheap_duplicates_match_multiset_oracle():
    """Where the reference's tie bug fires (duplicate keys), the oracle still
    returns the k smallest at every delete."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        k = 1 << int(rng.integers(0, 5))
        h = O.SeqHeap(trial % 2, k, 4096, True)
        ms = SortedList()
        for _ in range(200):
            if rng.integers(0, 2):
                n = k if rng.integers(0, 4) else int(rng.integers(1, k + 1))
                keys = rng.integers(0, 12, size=n).astype(np.uint64)
                assert h.insert(keys) == 0
                ms.update(keys.tolist())
            else:
                st, got = h.delete_min()
                exp = [ms.pop(0) for _ in range(min(k, len(ms)))]
                assert got.tolist() == exp


def test_seqheap_capacity_and_errors():
    h = O.SeqHeap(0, 2, 2)
    assert h.insert(np.array([1, 2], np.uint64)) == 0
    assert h.insert(np.array([3, 4], np.uint64)) == 0
    assert h.insert(np.array([5, 6], np.uint64)) == O.E_CAPACITY
    assert h.insert(np.array([9], np.uint64)) == 0
    assert h.insert(np.array([2**64 - 1], np.uint64)) == O.E_INVALID_KEY


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
def test_seqheap_matches_reference_on_unique_keys_live():
    rng = np.random.default_rng(5)
    for trial in range(60):
        k = 1 << int(rng.integers(0, 6))
        var, elide = trial % 2, bool((trial // 2) % 2)
        h, r = O.SeqHeap(var, k, 4096, elide), O.RefHeap(var, k, 4096, elide)
        for _ in range(200):
            if rng.integers(0, 2) == 0:
                n = int(rng.integers(1, k + 1)) if rng.integers(0, 4) == 0 else k
                keys = rng.choice(1 << 40, n, replace=False).astype(np.uint64)
                assert h.insert(keys) == r.insert(keys)
            else:
                a, b = h.delete_min(), r.delete_min()
                assert a[0] == b[0] and a[1].tolist() == b[1].tolist()
        assert h.counters() == r.counters()


# ------------------------------------------------------------- apps -----
def test_dijkstra_small_grid_matches_reference():
    for case in golden("apps.json")["grid_small"]:
        off, nbr, w = O.grid_graph(case["rows"], case["cols"], case["seed"])
        d = O.dijkstra(off, nbr, w, case["source"])
        assert d.tolist() == case["dist"]


def test_grid_2048_source0_sum():
    g = golden("apps.json")["grid_2048"][0]
    off, nbr, w = O.grid_graph(2048, 2048, 1)
    assert nbr.size == 16769024
    d = O.dijkstra(off, nbr, w, g["source"])
    assert int(d.sum(dtype=np.uint64)) == g["sum"] == 2117861108318
    assert int(d.max()) == g["max"] == 943358


def test_knapsack_generator_and_dp():
    for case in golden("apps.json")["knapsack"]:
        if case["n"] * case["capacity"] > 2e7:
            continue
        w, b, cap = O.generate_knapsack(case["type"], case["n"], case["range"], case["seed"])
        assert cap == case["capacity"]
        assert w[:4].tolist() == case["w_head"] and b[:4].tolist() == case["b_head"]
        assert O.knapsack_dp(w, b, cap) == case["dp"]


def test_knapsack_appendix_b_optima():
    opt = {(c["type"], c["range"], c["seed"]): c["dp"] for c in golden("apps.json")["knapsack"]
           if c["n"] == 200}
    assert [opt[(0, 1000, s)] for s in (1, 2, 3)] == [64500, 64300, 64800]
    assert [opt[(3, 7000, s)] for s in (1, 2, 3)] == [350000, 350000, 350000]
    assert [opt[(1, 1000, s)] for s in (1, 2, 3)] == [64028, 64114, 64395]


# ---------------------------------------------------------- lincheck -----
def _op(opid, kind, keys, inv, acq, rel, res):
    r = LC.OpRecord(worker=opid, opid=opid, op=kind, keys=list(keys), invoke_ts=inv, respond_ts=res)
    r.locks = [LC.LockSpan(1, acq, rel)]
    r.root_acquire_ts, r.root_release_ts = acq, rel
    r.last_acquire_ts, r.last_release_ts = acq, rel
    return r


def test_lincheck_trivial_and_mutation():
    hist = [_op(0, LC.INSERT, [3], 1, 2, 3, 4), _op(1, LC.INSERT, [1], 5, 6, 7, 8),
            _op(2, LC.DELETE, [1], 9, 10, 11, 12), _op(3, LC.DELETE, [3], 13, 14, 15, 16)]
    assert LC.check_td(hist, 1).passed and LC.check_bu(hist, 1).passed
    assert LC.check_exhaustive(hist, 1).passed
    hist[2].keys, hist[3].keys = hist[3].keys, hist[2].keys
    assert not LC.check_td(hist, 1).passed
    assert not LC.check_exhaustive(hist, 1).passed


def test_lincheck_exhaustive_real_time_order():
    # delete returns a key whose insert starts after the delete responded
    hist = [_op(0, LC.DELETE, [1], 1, 2, 3, 4), _op(1, LC.INSERT, [1], 5, 6, 7, 8)]
    assert not LC.check_exhaustive(hist, 1).passed
    # overlapping ops commute
    hist = [_op(0, LC.DELETE, [1], 1, 6, 7, 9), _op(1, LC.INSERT, [1], 2, 3, 4, 5)]
    assert LC.check_exhaustive(hist, 1).passed


def test_lincheck_mutual_exclusion_and_order():
    a = _op(0, LC.INSERT, [1], 1, 2, 5, 9)
    b = _op(1, LC.INSERT, [2], 3, 4, 6, 10)
    ok, _ = LC.check_mutual_exclusion([a, b])
    assert not ok
    c = _op(2, LC.DELETE, [1], 1, 2, 8, 9)
    c.locks = [LC.LockSpan(3, 2, 7), LC.LockSpan(1, 3, 8)]
    ok, _ = LC.check_lock_order([c])
    assert not ok


def test_lock_order_refill_exception():
    """A refill span (the last node, EV_ACQ_REFILL) may overlap the same op's
    claim of one of its ancestors; any other descendant-first overlap fails."""
    c = _op(2, LC.DELETE, [1], 1, 2, 20, 21)
    # root, then the refill source 9 and its ancestor 2 (claimed while 9 is held)
    c.locks = [LC.LockSpan(1, 2, 19), LC.LockSpan(9, 3, 6, refill=True), LC.LockSpan(2, 4, 12)]
    assert LC.check_lock_order([c])[0]
    c.locks[1].refill = False
    assert not LC.check_lock_order([c])[0]
    # decode_history marks kind-4 acquisitions as refill spans
    ev = [dict(ts=1, op=0, kind=LC.EV_INV, node=0), dict(ts=2, op=0, kind=LC.EV_ACQ, node=1),
          dict(ts=3, op=0, kind=LC.EV_ACQ_REFILL, node=9), dict(ts=4, op=0, kind=LC.EV_ACQ, node=2),
          dict(ts=5, op=0, kind=LC.EV_REL, node=9), dict(ts=6, op=0, kind=LC.EV_REL, node=2),
          dict(ts=7, op=0, kind=LC.EV_REL, node=1), dict(ts=8, op=0, kind=LC.EV_RES, node=0)]
    (rec,) = LC.decode_history(ev, [LC.DELETE], [[1]])
    assert [s.refill for s in rec.locks] == [False, True, False]
    assert LC.check_lock_order([rec])[0]
