"""CPU suite: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/batchheap_b200.h declares; host-only entry points behave; the
product path refuses to run without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_1906_06504_b200 as P
from paper_1906_06504_b200 import _lib as L
from oracle import oracle as O

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "batchheap_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BH_API\s+[\w\s\*]+?\b(bh_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("bh_create", "bh_destroy", "bh_insert", "bh_delete_min", "bh_run_ops",
                 "bh_peek_stats", "bh_get_counters", "bh_check_invariants", "bh_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(L.LIB_PATH), "build() must produce the library"
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(bh_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the ctypes signature table covers them
    assert set(declared_symbols()) <= set(L.SIGNATURES)
    lib = L.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_bitrev_matches_oracle():
    for r in range(1, 5000):
        assert P.slot_for_rank(r) == O.slot_for_rank(r)
    assert [P.bit_reverse(c, 3) for c in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("bits", [32, 64])
def test_product_keygen_matches_oracle(bits):
    """The workload generator the bench uses (host C++ in the product
    library) reproduces generate_keys (proj/src/workload.cpp:162-180)."""
    got = P.generate_keys(1 << 16, 1, key_bits=bits)
    exp = O.generate_keys(1 << 16, 1)
    assert np.array_equal(got.astype(np.uint64), exp)
    assert P.generate_keys(10, 5, order=1).tolist() == list(range(10))
    assert P.generate_keys(4, 5, order=2).tolist() == [4, 3, 2, 1]


def test_phase_ops_plan():
    ops = P.phase_ops(0, 10, 4)
    assert ops["len"].tolist() == [4, 4, 2] and ops["offset"].tolist() == [0, 4, 8]
    ops = P.phase_ops(1, 10, 4)
    assert ops["kind"].tolist() == [1, 1, 1] and ops["offset"].tolist() == [0, 4, 8]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(P.DeviceError):
        P.GeneralizedHeap(P.Variant.TD, 4, 16)


def test_config_errors_are_raised_before_device_use():
    with pytest.raises(P.ConfigError):
        P.GeneralizedHeap(P.Variant.TD, 3, 16)
    with pytest.raises(P.ConfigError):
        P.GeneralizedHeap(P.Variant.TD, 4, 0)
    with pytest.raises(P.ConfigError):
        P.GeneralizedHeap(P.Variant.TD, 4, 16, key_bits=16)


@pytest.mark.gpu
def test_run_watchdog_reports_a_run_past_its_deadline():
    """bh_run_ops waits with a deadline (BH_RUN_TIMEOUT_S), the host half of
    the reference's deadlock watchdog (proj/src/workload.cpp:22-53): a run
    still going when it expires returns BH_E_INTERNAL instead of blocking."""
    import numpy as np
    from oracle import oracle as O
    from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops
    k, n = 1024, 1 << 22
    keys = O.generate_keys(n, 5).astype(np.uint32)
    heap = GeneralizedHeap(Variant.BU, k, n // k + 64, key_bits=32)
    old = os.environ.get("BH_RUN_TIMEOUT_S")
    os.environ["BH_RUN_TIMEOUT_S"] = "0.000001"
    try:
        with pytest.raises(Exception, match="watchdog"):
            heap.run_ops(phase_ops(0, n, k), keys, 0)
    finally:
        if old is None:
            del os.environ["BH_RUN_TIMEOUT_S"]
        else:
            os.environ["BH_RUN_TIMEOUT_S"] = old
    # the run itself finishes; the heap is whole afterwards
    d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
    out = d.out.reshape(-1, k)[np.argsort(d.seq, kind="stable")].reshape(-1).astype(np.uint64)
    assert np.array_equal(out, O.sort_u64(keys))
