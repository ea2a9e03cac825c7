"""History text format (proj/src/history.cpp) on the host: round trip,
parse/validate errors, and the reference's own History::parse + checker
accepting what paper_1906_06504_b200.history writes."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1906_06504_b200.history import History, InstrumentationError, OpKind, OpRecord


def sequential_history(variant, k, n_ops, seed):
    """A valid sequential history: ops one after another through the
    oracle's sequential heap, synthetic increasing timestamps."""
    rng = np.random.default_rng(seed)
    orc = O.SeqHeap(variant, k, 4 * n_ops + 8, True)
    ops, ts = [], 1
    for i in range(n_ops):
        if rng.integers(0, 3):
            keys = sorted(rng.integers(0, 1 << 30, size=int(rng.integers(1, k + 1))).tolist())
            orc.insert(np.array(keys, np.uint64))
            r = OpRecord(i, i, OpKind.Insert, keys)
        else:
            st, got = orc.delete_min()
            r = OpRecord(i, i, OpKind.Delete, [] if st == 3 else sorted(int(x) for x in got))
        r.invoke_ts, r.root_acquire_ts, r.root_release_ts = ts, ts + 1, ts + 2
        r.last_acquire_ts, r.last_release_ts, r.respond_ts = ts + 3, ts + 4, ts + 5
        ts += 6
        ops.append(r)
    return History(variant, k, ops)


@pytest.mark.parametrize("variant", [0, 1])
def test_round_trip(variant):
    h = sequential_history(variant, 4, 60, variant + 1)
    text = h.serialize()
    assert len(text.splitlines()) == h.event_count()
    h2 = History.parse(text, variant, 4)
    strip = lambda o: (o.worker, o.opid, o.op, o.keys, o.invoke_ts, o.respond_ts, o.root_acquire_ts,
                       o.root_release_ts)
    assert [strip(o) for o in h2.ops] == [strip(o) for o in h.ops]
    assert h2.serialize() == text


def test_parse_and_validate_errors():
    with pytest.raises(InstrumentationError):
        History.parse("1 0 0 inv ins 5\n2 0 0 bogus ins -\n", 0, 1)
    with pytest.raises(InstrumentationError):
        History.parse("1 0 0 inv ins 5\n", 0, 1)  # missing events
    bad = "1 0 0 inv ins 5\n3 0 0 acR ins -\n2 0 0 reR ins -\n4 0 0 res ins -\n"
    with pytest.raises(InstrumentationError):
        History.parse(bad, 0, 1)  # acR after reR


@pytest.mark.skipif(not os.path.exists(O.REF_HISTCHECK), reason="reference checker not built")
@pytest.mark.parametrize("variant", [0, 1])
def test_reference_parser_and_checker_accept_our_format(variant):
    h = sequential_history(variant, 4, 14, 7 + variant)
    r = O.ref_history_check(h.serialize(), variant, 4)
    assert r.get("pass") and r["overlap_ok"] and r["exhaustive"] == 1 and r["ops"] == 14, r
    # a corrupted result is rejected by the reference's checker
    for o in h.ops:
        if o.op == OpKind.Delete and o.keys:
            o.keys = [o.keys[0] + 1] + o.keys[1:]
            break
    r = O.ref_history_check(h.serialize(), variant, 4)
    assert r.get("pass") is False, r
