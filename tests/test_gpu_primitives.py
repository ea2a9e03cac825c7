"""Batch primitives on the GPU vs the oracle (reference batch_core KATs,
proj/tests/test_batch.cpp:32-113)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1906_06504_b200 import merge_split_device, sort_batches_device

pytestmark = pytest.mark.gpu

KS = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048]


def _dev(a: np.ndarray, bits: int) -> torch.Tensor:
    dt = torch.int32 if bits == 32 else torch.int64
    npdt = np.int32 if bits == 32 else np.int64
    return torch.from_numpy(a.astype(np.uint32 if bits == 32 else np.uint64).view(npdt).copy()).to("cuda")


def _host(t: torch.Tensor, bits: int) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32 if bits == 32 else np.uint64).astype(np.uint64)


def test_sort_kats():
    # sort_batch basics (test_batch.cpp:32-41): [5,1,3] -> [1,3,5]; [7] -> [7]
    for bits in (32, 64):
        rows = np.full((2, 4), 0, dtype=np.uint64)
        rows[0, :3] = [5, 1, 3]
        rows[1, :1] = [7]
        t = _dev(rows.ravel(), bits)
        lens = torch.tensor([3, 1], dtype=torch.int32, device="cuda")
        sort_batches_device(t.data_ptr(), 4, 2, bits, lens.data_ptr())
        torch.cuda.synchronize()
        got = _host(t, bits).reshape(2, 4)
        assert got[0, :3].tolist() == [1, 3, 5]
        assert got[1, :1].tolist() == [7]


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("k", KS)
def test_sort_matches_oracle(k, bits):
    rng = np.random.default_rng(k * 7 + bits)
    rows = 64
    hi = (1 << 32) - 1 if bits == 32 else (1 << 48)
    keys = rng.integers(0, hi, size=(rows, k), dtype=np.uint64)
    keys[::3] %= 7  # duplicate-heavy rows
    lens = rng.integers(1, k + 1, size=rows).astype(np.int32)
    lens[0] = k
    t = _dev(keys.ravel(), bits)
    lt = torch.from_numpy(lens).to("cuda")
    sort_batches_device(t.data_ptr(), k, rows, bits, lt.data_ptr())
    torch.cuda.synchronize()
    got = _host(t, bits).reshape(rows, k)
    for r in range(rows):
        n = int(lens[r])
        assert np.array_equal(got[r, :n], O.sort_u64(keys[r, :n])), r


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("k", KS)
def test_merge_matches_concat_sort_split(k, bits):
    # test_batch.cpp:65-81: merge_and_sort == sort(concat) split at k
    rng = np.random.default_rng(1000 + k + bits)
    pairs = 48
    rng_hi = 1000 if k > 4 else 40
    a = np.sort(rng.integers(0, rng_hi, size=(pairs, k), dtype=np.uint64), axis=1)
    b = np.sort(rng.integers(0, rng_hi, size=(pairs, k), dtype=np.uint64), axis=1)
    a[1] = np.arange(k)           # disjoint, ordered
    b[1] = np.arange(k) + k
    a[2] = np.arange(k) + k       # disjoint, swapped
    b[2] = np.arange(k)
    ta, tb = _dev(a.ravel(), bits), _dev(b.ravel(), bits)
    thi, tlo = torch.empty_like(ta), torch.empty_like(ta)
    merge_split_device(ta.data_ptr(), tb.data_ptr(), thi.data_ptr(), tlo.data_ptr(), k, pairs, bits)
    torch.cuda.synchronize()
    hi, lo = _host(thi, bits).reshape(pairs, k), _host(tlo, bits).reshape(pairs, k)
    for p in range(pairs):
        eh, el = O.merge_and_sort(a[p], b[p], k)
        assert np.array_equal(hi[p], eh) and np.array_equal(lo[p], el), p


def test_merge_kat():
    # test_batch.cpp:53-63: [1,3,5,7]+[2,4,6,8], k=4 -> hi [1,2,3,4], lo [5,6,7,8]
    for bits in (32, 64):
        ta = _dev(np.array([1, 3, 5, 7], dtype=np.uint64), bits)
        tb = _dev(np.array([2, 4, 6, 8], dtype=np.uint64), bits)
        thi, tlo = torch.empty_like(ta), torch.empty_like(ta)
        merge_split_device(ta.data_ptr(), tb.data_ptr(), thi.data_ptr(), tlo.data_ptr(), 4, 1, bits)
        torch.cuda.synchronize()
        assert _host(thi, bits).tolist() == [1, 2, 3, 4]
        assert _host(tlo, bits).tolist() == [5, 6, 7, 8]
