"""The device-specific fast paths against the reference-protocol paths they
replace (both are kept; debug flags select the reference one):

* BU climb under the phase gate (relaxed park, re-take without reload)
  vs the reference climb (kDbgParkClimb);
* insert combining in the root queue lock vs one root hold per insert
  (kDbgNoCombine);
* the split heapify schedule at every CTA width (K=64 runs one thread
  group, K>=128 two).
Sequential bulk runs (one CTA) must leave identical layouts; concurrent
runs must drain the sorted input."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops

from test_gpu_bulk import mixed_ops

pytestmark = pytest.mark.gpu
PARK_CLIMB = 0x1000
NO_COMBINE = 0x800


def drain(heap, n, k, bits=32):
    n_del = (n + k - 1) // k
    dt = np.uint32 if bits == 32 else np.uint64
    d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, dt), n_del * k)
    assert np.all(d.status == 0)
    order = np.argsort(d.seq, kind="stable")
    out = d.out.reshape(n_del, k)[order]
    lens = d.lens[order]
    return np.concatenate([out[i, :lens[i]] for i in range(n_del)]).astype(np.uint64)


@pytest.mark.parametrize("k", [4, 64, 1024])
def test_gated_climb_same_layout_as_reference_climb(k):
    rng = np.random.default_rng(k)
    ops, pool, out_len, _ = mixed_ops(rng, 600, k, 20, 1 << 24)
    dumps = []
    for flags in (0, PARK_CLIMB):
        heap = GeneralizedHeap(Variant.BU, k, 700, debug_flags=flags)
        r = heap.run_ops(ops, pool, out_len, ctas=1)  # sequential: ticket order
        assert set(np.unique(r.status).tolist()) <= {0, 3}
        keys, part, states = heap.dump()
        results = [r.out[o["offset"]:o["offset"] + r.lens[i]].tolist() for i, o in enumerate(ops) if o["kind"] == 1]
        dumps.append((keys.copy(), part.copy(), heap.counters().__dict__, results))
        assert heap.check_invariants().ok
    (k0, p0, c0, o0), (k1, p1, c1, o1) = dumps
    assert np.array_equal(k0, k1) and np.array_equal(p0, p1)
    assert c0 == c1
    assert o0 == o1


@pytest.mark.parametrize("k", [64, 1024])
@pytest.mark.parametrize("flags", [0, PARK_CLIMB, NO_COMBINE, PARK_CLIMB | NO_COMBINE])
def test_concurrent_phase_drain_all_path_combinations(k, flags):
    n = (1 << 18) + 3 * k // 2 + 1
    keys = O.generate_keys(n, 7)
    heap = GeneralizedHeap(Variant.BU, k, n // k + 200, key_bits=32, debug_flags=flags)
    ins = heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
    assert np.all(ins.status == 0)
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    assert np.array_equal(drain(heap, n, k), O.sort_u64(keys))


def test_combining_serves_waiters():
    """Full-batch BU inserts from many CTAs: most are served by a combiner."""
    k, n = 256, 1 << 20
    keys = O.generate_keys(n, 3)
    heap = GeneralizedHeap(Variant.BU, k, n // k + 200, key_bits=32, profile=True)
    heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
    p = heap.profile()
    assert p["served"] > 0 and p["serve_holds"] > 0
    assert p["ins_ops"] == n // k  # every insert counted once, served or not
    assert np.array_equal(drain(heap, n, k), O.sort_u64(keys))


@pytest.mark.parametrize("k", [64, 128, 256])
def test_split_schedule_widths_mixed_td(k):
    rng = np.random.default_rng(99 + k)
    ops, pool, out_len, _ = mixed_ops(rng, 3000, k, 20, 1 << 16)
    heap = GeneralizedHeap(Variant.TD, k, 3100)
    r = heap.run_ops(ops, pool, out_len)
    assert set(np.unique(r.status).tolist()) <= {0, 3}
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    deleted = np.concatenate([r.out[o["offset"]:o["offset"] + r.lens[i]]
                              for i, o in enumerate(ops) if o["kind"] == 1] + [np.zeros(0, np.uint64)])
    acc = np.sort(np.concatenate([deleted.astype(np.uint64), heap.collect_resident()]))
    assert np.array_equal(acc, O.sort_u64(pool))


@pytest.mark.skipif(not __import__("os").path.exists(O.REF_HISTCHECK), reason="reference checker not built")
@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
@pytest.mark.parametrize("key_hi", [12, 1 << 40])
def test_device_history_passes_reference_checker(variant, key_hi):
    """A recorded concurrent device run, written in the reference's history
    text format by paper_1906_06504_b200.history, is accepted by the
    reference's own History::parse and check_td / check_bu (and, for BU, its
    overlap-window scan); small histories also by check_exhaustive."""
    from paper_1906_06504_b200.history import History, history_of
    for trial in range(4):
        rng = np.random.default_rng(500 + trial + int(variant) * 10 + (key_hi & 7))
        k = 2 if key_hi == 12 else 8
        n_ops = 14 if trial == 0 else 400
        ops, pool, out_len, _ = mixed_ops(rng, n_ops, k, 25, key_hi)
        heap = GeneralizedHeap(variant, k, n_ops + 8, record=True)
        r = heap.run_ops(ops, pool, out_len, ctas=64)
        h = history_of(heap, ops, r, pool)
        text = h.serialize()
        assert History.parse(text, int(variant), k).serialize() == text
        res = O.ref_history_check(text, int(variant), k)
        assert res.get("pass") and res["overlap_ok"], res
        if len(h.ops) <= 16:
            assert res["exhaustive"] == 1, res
