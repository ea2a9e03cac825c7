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
