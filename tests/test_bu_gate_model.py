"""The BU phase gate, on the random-interleaving model of the reference's BU
protocol (tools/sim_bu.py: proj/src/heap.cpp:123-188, 295-407, 420-531,
547-667 step for step, every shared access a scheduling point, k=1).

Without the gate, some schedules end with a quiescent heap that breaks
property 1 (a climber's parked slot taken over by a deleter, INSHOLD ->
DELMOD, heap.cpp:508-516,567-573, then consumed by another climber's parent
claim); the seeds below are such schedules.  With the gate (a climb and a
delete heapify never overlap, DESIGN.md section 4 item 2), the same workloads
and hundreds of other schedules keep properties 1-3 and the key multiset.
CPU only."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import sim_bu  # noqa: E402

BROKEN_WITHOUT_GATE = [2120, 2703, 2747, 3161]  # found by scanning seeds 0..3999


@pytest.fixture
def model():
    saved = (sim_bu.GATE, sim_bu.TAGS, sim_bu.RECHECK)
    yield sim_bu
    sim_bu.GATE, sim_bu.TAGS, sim_bu.RECHECK = saved


def test_reference_bu_breaks_property1_without_gate(model):
    model.GATE = False
    for seed in BROKEN_WITHOUT_GATE:
        bad, multiset_ok = model.run(seed)
        assert bad or not multiset_ok, seed
        assert any(kind == "prop1" for kind, _ in bad) or not multiset_ok, (seed, bad)


def test_phase_gate_keeps_invariants(model):
    model.GATE = True
    for seed in BROKEN_WITHOUT_GATE + list(range(600)):
        bad, multiset_ok = model.run(seed)
        assert not bad and multiset_ok, (seed, bad[:5])


@pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["ref_available"]).ref_available(),
                    reason="reference library (oracle/_ref) not built")
def test_reference_bu_fails_its_own_check_bu_at_64_threads():
    """The unmodified reference BU heap (oracle/_ref) under its own stress
    runner (proj/src/workload.cpp:75-147) with 64 worker threads and unique
    keys: the quiescent invariants and the multiset hold, but its own
    constructive check_bu (proj/src/lincheck.cpp:73-86) rejects the
    recorded histories -- the overlap of climbs and delete heapifies that
    the phase gate removes from the CUDA heap."""
    import ctypes as C
    from oracle import oracle as O
    r = O.ref()
    r.ref_stress.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                             C.c_uint64, C.c_int, C.POINTER(C.c_int)]
    out = (C.c_int * 6)()
    rejected = 0
    for seed in range(10):
        assert r.ref_stress(1, 8, 64, 200, 25, seed, 1 << 40, 1, out) == 0
        assert out[0] and out[1], list(out)  # invariants, multiset
        rejected += out[2] == 0
    assert rejected > 0
