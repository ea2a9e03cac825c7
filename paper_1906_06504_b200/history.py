"""Concurrent-execution histories of the device heap, in the reference's
model and text format (proj/include/batchheap/history.hpp,
proj/src/history.cpp, proj/src/instrumentation.cpp).

A heap created with ``record=True`` (BH_FLAG_RECORD) logs, per operation,
invoke / respond and every lock acquire / release against one global device
clock (``bh_history``).  ``history_from_run`` folds that log into
``OpRecord``s the way ``Recorder`` does (root window = the first span on
node 1; last-lock window = the span released last), and ``History``
serializes to / parses from the reference's line format

    ts worker opid kind op key1,key2,...

kind in {inv, res, acR, reR, acL, reL}; op in {ins, del}; "-" for no keys;
TD histories carry 4 events per op, BU ones add acL/reL for inserts
(history.cpp:56-84).  A serialized device history is therefore readable by
the reference's own ``History::parse`` and checkers.  The worker field is
the op index (each op ran on its own CTA turn).
"""
from __future__ import annotations

import dataclasses
import enum
from typing import Dict, List, Sequence

import numpy as np

EV_INV, EV_RES, EV_ACQ, EV_REL, EV_ACQ_REFILL = 0, 1, 2, 3, 4  # bh_event.kind (bh_internal.h EventKind)


class OpKind(enum.IntEnum):
    Insert = 0
    Delete = 1


class InstrumentationError(RuntimeError):
    """batchheap::InstrumentationError (history.hpp:32-34)."""


@dataclasses.dataclass
class LockSpan:
    node: int
    acquire_ts: int
    release_ts: int = 0


@dataclasses.dataclass
class OpRecord:
    """OpRecord (history.hpp:42-57)."""
    worker: int
    opid: int
    op: OpKind
    keys: List[int]
    invoke_ts: int = 0
    respond_ts: int = 0
    root_acquire_ts: int = 0
    root_release_ts: int = 0
    last_acquire_ts: int = 0
    last_release_ts: int = 0
    locks: List[LockSpan] = dataclasses.field(default_factory=list)


def _keys_field(keys: Sequence[int]) -> str:
    return ",".join(str(int(x)) for x in keys) if len(keys) else "-"


@dataclasses.dataclass
class History:
    """History (history.hpp:59-71): variant (0 TD, 1 BU), node capacity k, ops."""
    variant: int
    k: int
    ops: List[OpRecord]

    def event_count(self) -> int:  # history.cpp:47-54
        return sum(4 + (2 if self.variant == 1 and o.op == OpKind.Insert else 0) for o in self.ops)

    def serialize(self) -> str:  # history.cpp:56-84
        events = []
        for o in self.ops:
            ins = o.op == OpKind.Insert
            events.append((o.invoke_ts, o, "inv", o.keys if ins else []))
            events.append((o.root_acquire_ts, o, "acR", []))
            events.append((o.root_release_ts, o, "reR", []))
            if self.variant == 1 and ins:
                events.append((o.last_acquire_ts, o, "acL", []))
                events.append((o.last_release_ts, o, "reL", []))
            events.append((o.respond_ts, o, "res", [] if ins else o.keys))
        events.sort(key=lambda e: e[0])
        return "".join(f"{ts} {o.worker} {o.opid} {kind} {'ins' if o.op == OpKind.Insert else 'del'} "
                       f"{_keys_field(keys)}\n" for ts, o, kind, keys in events)

    @staticmethod
    def parse(text: str, variant: int, k: int) -> "History":  # history.cpp:86-131
        recs: Dict[tuple, OpRecord] = {}
        for n, line in enumerate(text.splitlines(), 1):
            if not line.strip():
                continue
            f = line.split()
            if len(f) != 6:
                raise InstrumentationError(f"history parse error at line {n}")
            ts, worker, opid, kind, op, kf = int(f[0]), int(f[1]), int(f[2]), f[3], f[4], f[5]
            r = recs.setdefault((worker, opid), OpRecord(worker, opid, OpKind.Insert, []))
            r.op = OpKind.Insert if op == "ins" else OpKind.Delete
            keys = [] if kf == "-" else [int(x) for x in kf.split(",")]
            if kind == "inv":
                r.invoke_ts = ts
                if r.op == OpKind.Insert:
                    r.keys = keys
            elif kind == "res":
                r.respond_ts = ts
                if r.op == OpKind.Delete:
                    r.keys = keys
            elif kind == "acR":
                r.root_acquire_ts = ts
            elif kind == "reR":
                r.root_release_ts = ts
            elif kind == "acL":
                r.last_acquire_ts = ts
            elif kind == "reL":
                r.last_release_ts = ts
            else:
                raise InstrumentationError(f"unknown event kind '{kind}' at line {n}")
        for r in recs.values():
            if r.last_release_ts == 0:
                r.last_acquire_ts, r.last_release_ts = r.root_acquire_ts, r.root_release_ts
        h = History(variant, k, sorted(recs.values(), key=lambda r: r.invoke_ts))
        h.validate()
        return h

    def validate(self) -> None:  # history.cpp:133-165
        seen = []
        for o in self.ops:
            where = f"op {o.opid} of worker {o.worker}"
            if 0 in (o.invoke_ts, o.respond_ts, o.root_acquire_ts, o.root_release_ts):
                raise InstrumentationError("missing event in " + where)
            if not (o.invoke_ts < o.root_acquire_ts < o.root_release_ts < o.respond_ts):
                raise InstrumentationError("event order violated in " + where)
            if not (o.invoke_ts < o.last_acquire_ts < o.last_release_ts < o.respond_ts):
                raise InstrumentationError("last-lock window invalid in " + where)
            for s in o.locks:
                if s.release_ts == 0 or s.acquire_ts >= s.release_ts:
                    raise InstrumentationError("unreleased lock in " + where)
            seen += [o.invoke_ts, o.respond_ts]
        if len(seen) != len(set(seen)):
            raise InstrumentationError("duplicate timestamps in history")


def history_from_run(events: np.ndarray, op_kinds: Sequence[int], op_keys: Sequence[Sequence[int]],
                     variant: int, k: int, skip=()) -> History:
    """Fold a device event log (``GeneralizedHeap.history_events()``) into a
    History the way Recorder::op_begin/lock_acquired/lock_released/op_end
    does (instrumentation.cpp:47-131).  ``op_keys[i]`` is op i's insert
    argument or delete result; ops in ``skip`` (failed: capacity, invalid
    key) and ops without events are left out, as Recorder::op_abort."""
    by_op: Dict[int, list] = {}
    for e in events:
        # the device clock starts at 0; the reference's at 1 (0 = "missing")
        by_op.setdefault(int(e["op"]), []).append((int(e["ts"]) + 1, int(e["kind"]), int(e["node"])))
    skip = set(skip)
    ops = []
    for i, evs in by_op.items():
        if i in skip:
            continue
        evs.sort()
        rec = OpRecord(i, i, OpKind(int(op_kinds[i])), sorted(int(x) for x in op_keys[i]))
        held: Dict[int, LockSpan] = {}
        for ts, kind, node in evs:
            if kind == EV_INV:
                rec.invoke_ts = ts
            elif kind == EV_RES:
                rec.respond_ts = ts
            elif kind in (EV_ACQ, EV_ACQ_REFILL):  # the text format has no refill mark
                if node in held:
                    raise InstrumentationError(f"op {i}: node {node} acquired twice")
                held[node] = LockSpan(node, ts)
            elif kind == EV_REL:
                span = held.pop(node, None)
                if span is None:
                    raise InstrumentationError(f"op {i}: release of node {node} without acquire")
                span.release_ts = ts
                rec.locks.append(span)
        if held:
            raise InstrumentationError(f"op {i}: lock never released")
        rec.locks.sort(key=lambda s: s.acquire_ts)
        root = [s for s in rec.locks if s.node == 1]
        if root:
            rec.root_acquire_ts, rec.root_release_ts = root[0].acquire_ts, root[0].release_ts
        last = max(rec.locks, key=lambda s: s.release_ts, default=None)
        if last is not None:
            rec.last_acquire_ts, rec.last_release_ts = last.acquire_ts, last.release_ts
        ops.append(rec)
    return History(variant, k, sorted(ops, key=lambda r: r.invoke_ts))


def history_of(heap, ops: np.ndarray, result, key_pool: np.ndarray) -> History:
    """The History of the last bulk run of a ``record=True`` heap:
    ``ops``/``key_pool`` as passed to ``run_ops`` and its ``RunResult``."""
    keys = []
    for i, o in enumerate(ops):
        if o["kind"] == 0:
            keys.append(key_pool[o["offset"]:o["offset"] + o["len"]].tolist())
        else:
            keys.append(result.out[o["offset"]:o["offset"] + result.lens[i]].tolist())
    skip = [i for i in range(len(ops)) if result.status[i] not in (0, 3)]
    return history_from_run(heap.history_events(), ops["kind"], keys, int(heap.variant), heap.node_capacity(),
                            skip)
