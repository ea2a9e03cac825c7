"""Bulk (persistent-kernel) runs on the GPU.

* Phase-separated workloads (BASELINE configs 1 and 2): insert-all then
  deleteMin-all must drain exactly sorted(input); checked against the oracle at
  2^20 and, at the full 2^26 size, against the reference's golden checksums
  (tests/golden/keygen.json).
* Mixed concurrent workloads (config 3): multiset conservation, quiescent
  invariants, and linearizability of the recorded device history
  (check_td / check_bu / mutual exclusion / lock order / Lemma 3.3).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import lincheck as LC
from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, HeapOptions, Variant, make_ops, phase_ops

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.abspath(__file__))


def phase_run(variant, k, n, bits, seed=1, ctas=0):
    keys = O.generate_keys(n, seed)
    dt = np.uint32 if bits == 32 else np.uint64
    heap = GeneralizedHeap(variant, k, n // k + 64 + 2, key_bits=bits)
    ins = heap.run_ops(phase_ops(0, n, k), keys.astype(dt), 0, ctas=ctas)
    assert np.all(ins.status == 0)
    n_del = (n + k - 1) // k
    dels = heap.run_ops(phase_ops(1, n, k), np.zeros(0, dt), n_del * k, ctas=ctas)
    assert np.all(dels.status == 0)
    # order the delete batches by their root-lock sequence (linearization order)
    order = np.argsort(dels.seq, kind="stable")
    out = dels.out.reshape(n_del, k)[order]
    lens = dels.lens[order]
    stream = np.concatenate([out[i, :lens[i]] for i in range(n_del)]).astype(np.uint64)
    return heap, keys, stream


@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
@pytest.mark.parametrize("bits", [32, 64])
def test_phase_2pow20_k1024_matches_oracle(variant, bits):
    heap, keys, stream = phase_run(variant, 1024, 1 << 20, bits)
    assert np.array_equal(stream, O.sort_u64(keys))
    g = json.load(open(os.path.join(ROOT, "golden", "keygen.json")))["20"]
    s, x, h = O.checksums(stream)
    assert (s, x, h) == (g["sum"], g["xor"], g["poly_hash"])
    assert heap.peek_stats().key_count == 0
    rep = heap.check_invariants()
    assert rep.ok, rep.detail


@pytest.mark.parametrize("k", [1, 2, 8, 32, 256, 512, 2048])
@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
def test_phase_k_sweep_small(k, variant):
    n = max(64 * k, 1 << 14) + 3 * k // 2 + 1  # ragged tail: last batch partial
    n = min(n, 1 << 18)
    heap, keys, stream = phase_run(variant, k, n, 32)
    assert np.array_equal(stream, O.sort_u64(keys))


@pytest.mark.slow
@pytest.mark.parametrize("k", [256, 512, 1024, 2048])
def test_phase_2pow26_golden(k):
    """BASELINE config 2 at full size: the drain equals the sorted input,
    checked through the reference's golden fingerprints (sum, xor, polynomial
    hash of the sorted stream) plus sortedness."""
    n = 1 << 26
    dev = torch.device("cuda")
    keys = O.generate_keys(n, 1).astype(np.uint32)
    heap = GeneralizedHeap(Variant.BU, k, n // k + 1024, key_bits=32)
    pool = torch.from_numpy(keys.view(np.int32)).to(dev)
    n_ops = n // k
    ops_i = torch.from_numpy(phase_ops(0, n, k).view(np.uint8)).to(dev)
    ops_d = torch.from_numpy(phase_ops(1, n, k).view(np.uint8)).to(dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.empty(n_ops, dtype=torch.int32, device=dev)
    seq = torch.empty(n_ops, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    heap.run_ops_ptr(ops_i.data_ptr(), n_ops, pool.data_ptr(), 0, st.data_ptr(), 0, 0, stream=s)
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0
    heap.run_ops_ptr(ops_d.data_ptr(), n_ops, 0, out.data_ptr(), st.data_ptr(), 0, seq.data_ptr(), stream=s)
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0
    order = torch.argsort(seq)
    stream = out.view(n_ops, k)[order].reshape(-1).cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.all(stream[:-1] <= stream[1:])
    g = json.load(open(os.path.join(ROOT, "golden", "keygen.json")))["26"]
    assert O.checksums(stream) == (g["sum"], g["xor"], g["poly_hash"])
    assert heap.peek_stats().key_count == 0


def mixed_ops(rng, n_ops, k, partial_pct, key_hi, pre_nodes=0):
    kinds, lens, offs, pool = [], [], [], []
    out_at = 0
    for i in range(pre_nodes):
        pool.append(rng.integers(0, key_hi, size=k, dtype=np.uint64))
    pre_pool = np.concatenate(pool) if pool else np.zeros(0, np.uint64)
    at = pre_pool.size
    chunks = [pre_pool]
    for _ in range(n_ops):
        if rng.integers(0, 2) == 0:
            n = k if (k == 1 or rng.integers(0, 100) >= partial_pct) else int(rng.integers(1, k))
            chunks.append(rng.integers(0, key_hi, size=n, dtype=np.uint64))
            kinds.append(0); lens.append(n); offs.append(at)
            at += n
        else:
            kinds.append(1); lens.append(0); offs.append(out_at)
            out_at += k
    return make_ops(kinds, lens, offs), np.concatenate(chunks), out_at, pre_pool


@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
@pytest.mark.parametrize("k", [1, 4, 16, 64, 128, 256, 1024, 2048])
def test_mixed_concurrent_multiset_and_invariants(variant, k):
    """SPEC acceptance 1 analogue: 50/50 ins/del, 20% partial batches, many
    CTAs at once; quiescent properties 1-3 and multiset conservation."""
    rng = np.random.default_rng(k + 17 * int(variant))
    n_ops = 4000 if k < 1024 else 1500
    ops, pool, out_len, _ = mixed_ops(rng, n_ops, k, 20, 1 << 20)
    heap = GeneralizedHeap(variant, k, n_ops + 8)
    r = heap.run_ops(ops, pool, out_len)
    assert set(np.unique(r.status).tolist()) <= {0, 3}
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    deleted = np.concatenate([r.out[o["offset"]:o["offset"] + r.lens[i]]
                              for i, o in enumerate(ops) if o["kind"] == 1] + [np.zeros(0, np.uint64)])
    acc = np.sort(np.concatenate([deleted.astype(np.uint64), heap.collect_resident()]))
    assert np.array_equal(acc, O.sort_u64(pool))
    # sorted drain from quiescence
    drained = []
    while (b := heap.try_delete_min()) is not None:
        drained.extend(b.tolist())
    assert drained == sorted(drained)


def _recorded_history(heap, ops, r, pool):
    ev = heap.history_events()
    keys = []
    for i, o in enumerate(ops):
        if o["kind"] == 0:
            keys.append(pool[o["offset"]:o["offset"] + o["len"]].tolist())
        else:
            keys.append(r.out[o["offset"]:o["offset"] + r.lens[i]].tolist())
    skip = {i for i in range(len(ops)) if r.status[i] not in (0, 3)}
    return LC.decode_history(ev, ops["kind"], keys, skip)


@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
@pytest.mark.parametrize("key_hi", [12, 1 << 40])
def test_linearizability_recorded(variant, key_hi):
    """SPEC acceptance 3/5 analogue: device event log of a concurrent run
    passes the constructive checker of its variant, mutual exclusion and lock
    order; BU runs also satisfy the Lemma 3.3 window scan."""
    for trial in range(6):
        rng = np.random.default_rng(trial * 101 + int(variant) + (key_hi & 0xFF))
        k = 2 if key_hi == 12 else 8
        ops, pool, out_len, _ = mixed_ops(rng, 600, k, 25, key_hi)
        heap = GeneralizedHeap(variant, k, 700, record=True)
        r = heap.run_ops(ops, pool, out_len, ctas=64)
        hist = _recorded_history(heap, ops, r, pool)
        assert LC.validate(hist) is None
        ok, why = LC.check_mutual_exclusion(hist)
        assert ok, why
        ok, why = LC.check_lock_order(hist)
        assert ok, why
        # the reference's constructive orders: TD by root release, BU by
        # last-lock release (proj/src/lincheck.cpp:53-86) ...
        res = LC.check_td(hist, k) if variant == Variant.TD else LC.check_bu(hist, k)
        assert res.passed, res.detail
        # ... and the just-in-time witness builder agrees
        jit = LC.check_jit(hist, k)
        assert jit.passed, jit.detail
        if variant == Variant.BU:
            ok, why = LC.check_bu_overlap_windows(hist)
            assert ok, why
        rep = heap.check_invariants()
        assert rep.ok, rep.detail


@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
def test_constructive_implies_exhaustive(variant):
    """SPEC acceptance 4 analogue on small histories (<= 16 ops)."""
    for trial in range(200):
        rng = np.random.default_rng(5000 + trial)
        ops, pool, out_len, _ = mixed_ops(rng, 14, 2, 30, 12)
        heap = GeneralizedHeap(variant, 2, 32, record=True)
        r = heap.run_ops(ops, pool, out_len, ctas=4)
        hist = _recorded_history(heap, ops, r, pool)
        res = LC.check_td(hist, 2) if variant == Variant.TD else LC.check_bu(hist, 2)
        ex = LC.check_exhaustive(hist, 2)
        assert ex.passed, ex.detail
        # constructive PASS must imply exhaustive PASS (it produced a witness)
        assert res.passed, res.detail


def test_mutated_history_fails():
    """Swapping two delete results must be rejected (lincheck mutation test,
    proj/tests/test_lincheck.cpp:116-143)."""
    rng = np.random.default_rng(77)
    ops, pool, out_len, _ = mixed_ops(rng, 200, 4, 0, 1 << 30)
    heap = GeneralizedHeap(Variant.TD, 4, 256, record=True)
    r = heap.run_ops(ops, pool, out_len, ctas=16)
    hist = _recorded_history(heap, ops, r, pool)
    assert LC.check_td(hist, 4).passed
    dels = [h for h in hist if h.op == LC.DELETE and h.keys]
    assert len(dels) >= 2
    dels[0].keys, dels[-1].keys = dels[-1].keys, dels[0].keys
    assert not LC.check_td(hist, 4).passed


def test_ins_del_pairs_preseeded():
    """Config 3 shape: pre-seeded heap (initial levels) then ins-del pairs."""
    k = 1024
    rng = np.random.default_rng(3)
    levels = 8
    pre_nodes = (1 << levels) - 1
    pre = rng.integers(0, (1 << 32) - 1, size=pre_nodes * k, dtype=np.uint64)
    heap = GeneralizedHeap(Variant.BU, k, pre_nodes + 4096, key_bits=32)
    heap.run_ops(phase_ops(0, pre.size, k), pre.astype(np.uint32), 0)
    pairs = 2048
    pool = rng.integers(0, (1 << 32) - 1, size=pairs * k, dtype=np.uint64)
    kinds = np.tile([0, 1], pairs)
    lens = np.tile([k, 0], pairs)
    offs = np.empty(2 * pairs, np.uint64)
    offs[0::2] = np.arange(pairs) * k
    offs[1::2] = np.arange(pairs) * k
    r = heap.run_ops(make_ops(kinds, lens, offs), pool.astype(np.uint32), pairs * k)
    assert np.all(r.status == 0)
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    acc = np.sort(np.concatenate([r.out.astype(np.uint64), heap.collect_resident()]))
    assert np.array_equal(acc, np.sort(np.concatenate([pre, pool])))
