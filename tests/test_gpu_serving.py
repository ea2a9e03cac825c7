"""Delete serving (bh_heap.cuh serve_deletes): a delete holding the root
with deletes queued behind it runs their levels 0-1 from shared memory and
hands each continuation to the next waiter.  Compared with the one-root-hold-
per-delete path (kDbgNoDelServe): the same deleted batches in the same order
(each op still linearizes at its root step, in queue order), a valid heap
after a partial phase (properties 1-2, multiset), and a heap that keeps
working for later inserts and deletes."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, make_ops, phase_ops

pytestmark = pytest.mark.gpu
NO_DEL_SERVE = 0x2000


def _deleted(heap, n_ops, k):
    d = heap.run_ops(phase_ops(1, n_ops * k, k), np.zeros(0, np.uint32), n_ops * k)
    assert np.all(d.status == 0)
    order = np.argsort(d.seq, kind="stable")
    out = d.out.reshape(n_ops, k)[order]
    lens = d.lens[order]
    return np.concatenate([out[i, :lens[i]] for i in range(n_ops)]).astype(np.uint64)


@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
@pytest.mark.parametrize("k", [256, 1024, 2048])
def test_serving_engages_and_drains_sorted(k, variant):
    n = 1 << 20
    keys = O.generate_keys(n, 11)
    served = {}
    for flags in (0, NO_DEL_SERVE):
        heap = GeneralizedHeap(variant, k, n // k + 64, key_bits=32, profile=True, debug_flags=flags)
        assert np.all(heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0).status == 0)
        heap.profile(reset=True)
        got = _deleted(heap, n // k, k)
        served[flags] = heap.profile()["del_served"]
        assert np.array_equal(got, O.sort_u64(keys))
        assert heap.peek_stats().node_count == 0
        heap.close()
    assert served[0] > (n // k) // 2  # most deletes were served
    assert served[NO_DEL_SERVE] == 0


@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
@pytest.mark.parametrize("k", [256, 1024])
def test_serving_partial_phase_leaves_a_valid_heap(k, variant):
    n = (1 << 19) + 5 * k
    keys = O.generate_keys(n, 12).astype(np.uint64)
    heap = GeneralizedHeap(variant, k, 2 * (n // k) + 64, key_bits=32)
    assert np.all(heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0).status == 0)
    m = (n // k) // 2
    srt = np.sort(keys)
    assert np.array_equal(_deleted(heap, m, k), srt[:m * k])
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    assert np.array_equal(np.sort(heap.collect_resident().astype(np.uint64)), srt[m * k:])
    # the heap keeps working: more inserts, then the whole drain
    more = O.generate_keys(64 * k, 13).astype(np.uint64)
    ins = heap.run_ops(phase_ops(0, more.size, k), more.astype(np.uint32), 0)
    assert np.all(ins.status == 0)
    rest = np.sort(np.concatenate([srt[m * k:], more]))
    assert np.array_equal(_deleted(heap, rest.size // k, k), rest)


@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
def test_serving_with_interleaved_inserts_conserves_keys(variant):
    """Delete runs broken by inserts (BU phase gate included): servers stop at an insert in the queue;
    every key inserted comes out once, invariants hold at quiescence."""
    k, n = 1024, 1 << 19
    keys = O.generate_keys(2 * n, 14).astype(np.uint64)
    heap = GeneralizedHeap(variant, k, 2 * (2 * n // k) + 64, key_bits=32)
    assert np.all(heap.run_ops(phase_ops(0, n, k), keys[:n].astype(np.uint32), 0).status == 0)
    # 3 deletes, 1 insert, repeated
    n_ins = (n // k) // 2
    kinds, lens, offs = [], [], []
    di = 0
    for i in range(n_ins):
        for _ in range(3):
            kinds.append(1)
            lens.append(0)
            offs.append(di * k)
            di += 1
        kinds.append(0)
        lens.append(k)
        offs.append(n + i * k)
    ops = make_ops(np.array(kinds, np.uint32), np.array(lens, np.uint32), np.array(offs, np.uint64))
    r = heap.run_ops(ops, keys.astype(np.uint32), di * k)
    assert set(np.unique(r.status).tolist()) <= {0, 3}
    rep = heap.check_invariants()
    assert rep.ok, rep.detail
    out = [r.out[o["offset"]:o["offset"] + r.lens[i]] for i, o in enumerate(ops) if o["kind"] == 1]
    got = np.sort(np.concatenate(out + [heap.collect_resident()]).astype(np.uint64))
    assert np.array_equal(got, np.sort(keys[:n + n_ins * k]))


def test_serving_stays_within_its_launch():
    """Two delete launches on two streams share the root queue: a server
    must serve only ops of its own launch (their ops, out_pool and status
    arrays).  Ordered by their delete sequence, the two launches' batches
    together are the sorted prefix of the heap."""
    import torch

    k, n, m = 256, 1 << 19, 600
    keys = O.generate_keys(n, 21).astype(np.uint64)
    heap = GeneralizedHeap(Variant.BU, k, n // k + 64, key_bits=32)
    assert np.all(heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0).status == 0)
    dev = torch.device("cuda", 0)
    runs = []
    for _ in range(2):
        ops = torch.from_numpy(phase_ops(1, m * k, k).view(np.uint8)).to(dev)
        runs.append(dict(ops=ops, out=torch.zeros(m * k, dtype=torch.int32, device=dev),
                         st=torch.full((m,), 99, dtype=torch.int32, device=dev),
                         ln=torch.zeros(m, dtype=torch.int32, device=dev),
                         sq=torch.zeros(m, dtype=torch.int64, device=dev), stream=torch.cuda.Stream(dev)))
    torch.cuda.synchronize(dev)
    ctas = max(heap.max_ctas // 2, 2)
    for r in runs:
        heap.run_ops_ptr(r["ops"].data_ptr(), m, 0, r["out"].data_ptr(), r["st"].data_ptr(), r["ln"].data_ptr(),
                         r["sq"].data_ptr(), ctas=ctas, stream=r["stream"].cuda_stream)
    torch.cuda.synchronize(dev)
    seqs, batches = [], []
    for r in runs:
        st = r["st"].cpu().numpy()
        assert np.all(st == 0), np.unique(st)
        assert np.all(r["ln"].cpu().numpy() == k)
        out = r["out"].cpu().numpy().view(np.uint32).reshape(m, k).astype(np.uint64)
        seqs.append(r["sq"].cpu().numpy())
        batches.append(out)
    seq = np.concatenate(seqs)
    allb = np.concatenate(batches)[np.argsort(seq, kind="stable")]
    assert np.array_equal(np.sort(seq), np.arange(2 * m))
    assert np.array_equal(allb.reshape(-1), np.sort(keys)[:2 * m * k])
    rep = heap.check_invariants()
    assert rep.ok, rep.detail


@pytest.mark.parametrize("variant", [Variant.BU, Variant.TD])
def test_served_deletes_recorded_history_is_linearizable(variant):
    """Recorded heaps serve deletes too: each served op's root window and
    its node 1-3 spans are logged inside the server's hold, its lower lock
    events and response by the CTA that runs its continuation.  The history
    passes the same checkers as unserved runs."""
    from oracle import lincheck as LC
    from test_gpu_bulk import _recorded_history

    k = 256
    rng = np.random.default_rng(31 + int(variant))
    chunks, kinds, lens, offs = [], [], [], []
    at = out_at = 0
    plan = [0] * 200 + [1] * 100 + [int(x) for x in rng.integers(0, 2, size=60)]
    for kind in plan:
        if kind == 0:
            chunks.append(rng.integers(0, 1 << 40, size=k, dtype=np.uint64))
            kinds.append(0); lens.append(k); offs.append(at)
            at += k
        else:
            kinds.append(1); lens.append(0); offs.append(out_at)
            out_at += k
    ops = make_ops(np.array(kinds, np.uint32), np.array(lens, np.uint32), np.array(offs, np.uint64))
    pool = np.concatenate(chunks)
    served = 0
    for trial in range(4):
        heap = GeneralizedHeap(variant, k, 600, record=True, profile=True)
        r = heap.run_ops(ops, pool, out_at, ctas=12)  # the delete block queues up
        assert set(np.unique(r.status).tolist()) <= {0, 3}
        served += heap.profile()["del_served"]
        hist = _recorded_history(heap, ops, r, pool)
        assert LC.validate(hist) is None
        ok, why = LC.check_mutual_exclusion(hist)
        assert ok, why
        ok, why = LC.check_lock_order(hist)
        assert ok, why
        res = LC.check_td(hist, k) if variant == Variant.TD else LC.check_bu(hist, k)
        assert res.passed, res.detail
        jit = LC.check_jit(hist, k)
        assert jit.passed, jit.detail
        rep = heap.check_invariants()
        assert rep.ok, rep.detail
        heap.close()
    assert served > 0  # the history covered served deletes
