"""Random-interleaving model of the reference BU protocol (k=1), step for
step as proj/src/heap.cpp writes it (insert :123-188 + insert_bu :295-407,
do_delete :420-465 + refill :467-531 + heapify :547-667).  Every shared
read, CAS and write is a scheduling point.  Checks property 1 and multiset
conservation at quiescence.  Diagnostic only (tests/test_bu_gate_model.py
runs it).

GATE=True adds the BU phase gate of the CUDA heap (bh_heap.cuh gate_try /
gate_wait, DESIGN.md section 4 item 2) in its simplest form: under the root
lock, an insert that will climb (rank >= 2) waits while a delete heapify is
in flight, and a delete that will heapify (>= 2 nodes) waits while a climb is
in flight; a waiter lets the root go and queues again."""
import random
import sys

AVAIL, INUSE, TARGET, MARKED, INSHOLD, DELMOD = range(6)
SENT = float("inf")


TAGS = True
RECHECK = True
GATE = False


def S(v):
    return v & 7


class Heap:
    def __init__(self, slots):
        self.slots = slots
        self.st = [AVAIL] * (slots + 1)
        self.nd = [SENT] * (slots + 1)
        self.count = 0
        self.climbers = 0
        self.deleters = 0

    def cas(self, i, exp, new):
        if self.st[i] == exp or (not TAGS and S(self.st[i]) == S(exp) and exp < 8):
            self.st[i] = new
            return True
        return False


def slot_for_rank(r):
    lvl = r.bit_length() - 1
    base = 1 << lvl
    off = r - base
    rev = int(format(off, f"0{lvl}b")[::-1], 2) if lvl else 0
    return base + rev


def lock_avail(h, i):
    while True:
        yield
        if h.cas(i, AVAIL, INUSE):
            return


_tag = [0]


def gated(h, body, climb):
    """Run an op body behind the phase gate (root taken here)."""
    while True:
        yield from lock_avail(h, 1)
        yield
        needs = (h.count + 1 >= 2) if climb else (h.count >= 2)
        other = h.deleters if climb else h.climbers
        if needs and other > 0:
            yield
            h.st[1] = AVAIL
            continue
        break
    if needs:
        if climb:
            h.climbers += 1
        else:
            h.deleters += 1
    yield from body
    if needs:
        if climb:
            h.climbers -= 1
        else:
            h.deleters -= 1


def insert(h, key, log, root_held=False):
    if GATE and not root_held:
        yield from gated(h, insert(h, key, log, True), True)
        return
    _tag[0] += 1
    tag = _tag[0] if TAGS else 0
    if not root_held:
        yield from lock_avail(h, 1)
    yield
    rank = h.count + 1
    h.count = rank
    if rank == 1:
        yield
        h.nd[1] = key
        yield
        h.st[1] = AVAIL
        return
    target = slot_for_rank(rank)
    while True:
        yield
        s = h.st[target]
        if s == AVAIL and h.cas(target, AVAIL, INUSE):
            break
        if S(s) == DELMOD and h.cas(target, s, INUSE):
            break
    yield
    h.nd[target] = key
    yield
    h.st[1] = AVAIL
    cur = target
    while cur != 1:
        parent = cur // 2
        yield
        h.st[cur] = tag * 8 + INSHOLD
        while True:
            yield
            s = h.st[parent]
            if s == AVAIL and h.cas(parent, AVAIL, INUSE):
                break
            if S(s) == DELMOD and h.cas(parent, s, INUSE):
                break
        yield
        if h.nd[parent] == SENT:
            yield
            h.st[parent] = AVAIL
            while True:  # abandon_park
                yield
                s = h.st[cur]
                if s == tag * 8 + DELMOD or (not TAGS and S(s) == DELMOD):
                    if h.cas(cur, s, AVAIL):
                        return
                elif S(s) != INUSE:
                    return
        owned = False
        relock = False
        while True:
            yield
            s = h.st[cur]
            if s == tag * 8 + INSHOLD:
                if h.cas(cur, s, INUSE):
                    owned = True
                    break
            elif RECHECK and (s == AVAIL or S(s) == DELMOD):
                if h.cas(cur, s, INUSE):
                    relock = True  # not ours any more, but re-check it
                    break
            elif s == tag * 8 + DELMOD:
                if h.cas(cur, s, AVAIL):
                    break
            elif S(s) != INUSE:
                break  # consumed: AVAIL, or another climber's park / marker
        if relock:
            yield
            c, p = h.nd[cur], h.nd[parent]
            if c != SENT and c < p:
                yield
                h.nd[parent], h.nd[cur] = c, p
            yield
            h.st[cur] = AVAIL
        if owned:
            yield
            c, p = h.nd[cur], h.nd[parent]
            if c >= p:
                yield
                h.st[cur] = AVAIL
                yield
                h.st[parent] = AVAIL
                return
            yield
            h.nd[parent], h.nd[cur] = c, p
            yield
            h.st[cur] = AVAIL
        cur = parent
    yield
    h.st[1] = AVAIL


def acquire_child(h, slot):
    if slot > h.slots:
        return (slot, False, True, AVAIL)
    rel = AVAIL
    while True:
        yield
        s = h.st[slot]
        if s == AVAIL:
            if h.cas(slot, AVAIL, INUSE):
                break
        elif S(s) == INSHOLD:
            if h.cas(slot, s, INUSE):
                rel = (s & ~7) + DELMOD  # the marker keeps the owner's tag
                break
        elif S(s) == DELMOD:
            if h.cas(slot, s, INUSE):
                break
    yield
    return (slot, True, h.nd[slot] == SENT, rel)


def delete(h, log, root_held=False):
    if GATE and not root_held:
        yield from gated(h, delete(h, log, True), False)
        return
    if not root_held:
        yield from lock_avail(h, 1)
    yield
    nodes = h.count
    if nodes == 0:
        yield
        h.st[1] = AVAIL
        return
    yield
    log.append(h.nd[1])
    h.count = nodes - 1
    if nodes == 1:
        yield
        h.nd[1] = SENT
        yield
        h.st[1] = AVAIL
        return
    last = slot_for_rank(nodes)
    while True:
        yield
        s = h.st[last]
        if (s == AVAIL or S(s) == DELMOD) and h.cas(last, s, INUSE):
            rel = AVAIL
            break
        if S(s) == INSHOLD and h.cas(last, s, INUSE):
            rel = (s & ~7) + DELMOD
            break
    yield
    h.nd[1] = h.nd[last]
    yield
    h.nd[last] = SENT
    yield
    h.st[last] = rel
    cur, cur_rel = 1, AVAIL
    while True:
        l = yield from acquire_child(h, 2 * cur)
        r = yield from acquire_child(h, 2 * cur + 1)

        def release(c):
            if c[1]:
                h.st[c[0]] = c[3]
        if l[2] and r[2]:
            yield
            release(l)
            release(r)
            h.st[cur] = cur_rel
            return
        yield
        cmax = h.nd[cur]
        lmin = SENT if l[2] else h.nd[l[0]]
        rmin = SENT if r[2] else h.nd[r[0]]
        if cmax <= lmin and cmax <= rmin:
            yield
            release(l)
            release(r)
            h.st[cur] = cur_rel
            return
        if l[2]:
            hi, lo = r, l
        elif r[2]:
            hi, lo = l, r
        else:
            # k=1: batches never interleave; the smaller one is hi
            hi, lo = (l, r) if h.nd[l[0]] <= h.nd[r[0]] else (r, l)
        yield
        h.nd[cur], h.nd[hi[0]] = h.nd[hi[0]], h.nd[cur]
        yield
        release(lo)
        h.st[cur] = cur_rel
        cur, cur_rel = hi[0], hi[3]


def check(h):
    bad = []
    occupied = set(slot_for_rank(r) for r in range(1, h.count + 1))
    for s in range(1, h.slots + 1):
        if S(h.st[s]) != AVAIL:
            bad.append(("state", s))
        if s in occupied:
            if s > 1 and h.nd[s] < h.nd[s // 2]:
                bad.append(("prop1", s))
        elif h.nd[s] != SENT:
            bad.append(("unoccupied", s))
    return bad


def run(seed, workers=6, ops=40, slots=255):
    rng = random.Random(seed)
    h = Heap(slots)
    inserted, deleted = [], []
    keys = rng.sample(range(10**9), workers * ops)
    gens = []
    for w in range(workers):
        def worker(w=w):
            for i in range(ops):
                if rng.random() < 0.55:
                    k = keys[w * ops + i]
                    inserted.append(k)
                    yield from insert(h, k, deleted)
                else:
                    yield from delete(h, deleted)
        gens.append(worker())
    live = list(gens)
    while live:
        g = rng.choice(live)
        try:
            next(g)
        except StopIteration:
            live.remove(g)
    bad = check(h)
    resident = [h.nd[slot_for_rank(r)] for r in range(1, h.count + 1)]
    ms = sorted(inserted) == sorted(deleted + resident)
    return bad, ms


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    TAGS = "notags" not in sys.argv[2:]
    RECHECK = TAGS
    GATE = "gate" in sys.argv[2:]
    fails = 0
    for seed in range(n):
        bad, ms = run(seed)
        if bad or not ms:
            fails += 1
            if fails <= 3:
                print("seed", seed, "bad", bad[:5], "multiset ok" if ms else "MULTISET BROKEN")
    print(f"{fails} of {n} random schedules broke the quiescent invariants")
