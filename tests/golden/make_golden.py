"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libbatchheap_ref.so, built
by ``make -C oracle ref`` from /root/reference/proj/src) and records its
outputs.  Needs /root/reference at build time only; the fixtures are committed
and travel to the GPU box, the reference does not.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def keygen_fixture():
    r = O.ref()
    out = {}
    for log2n in (20, 26):
        n = 1 << log2n
        keys = np.empty(n, dtype=np.uint64)
        r.ref_generate_keys(0, n, 1, keys)
        s = np.sort(keys)
        total, xor, h = O.checksums(s)
        out[str(log2n)] = {
            "n": n, "seed": 1, "first": [int(v) for v in keys[:8]],
            "min": int(s[0]), "max": int(s[-1]), "sum": total, "xor": xor, "poly_hash": h,
            "adjacent_dups": int((s[1:] == s[:-1]).sum()),
            "count_u32_sentinel": int((keys == 0xFFFFFFFF).sum()),
        }
    for order in (1, 2):
        keys = np.empty(16, dtype=np.uint64)
        r.ref_generate_keys(order, 16, 3, keys)
        out["order%d" % order] = [int(v) for v in keys]
    return out


def heap_histories():
    """Single-threaded random op sequences run through the reference
    GeneralizedHeap.  Keys are drawn without replacement (the reference's
    equal-maxima tie bug needs duplicates), so these are
    exact for any correct implementation of the protocol, counters included."""
    rng = np.random.default_rng(20240611)
    cases = []
    for trial in range(48):
        k = int(2 ** (trial % 6))
        variant = (trial // 6) % 2
        elide = (trial // 12) % 2 == 0
        max_nodes = 256
        h = O.RefHeap(variant, k, max_nodes, elide)
        ops, args, results, statuses = [], [], [], []
        used = rng.choice(1 << 40, size=400 * k + 64, replace=False).astype(np.uint64)
        at = 0
        for step in range(160):
            if rng.integers(0, 3) != 0:
                n = k if rng.integers(0, 4) != 0 else int(rng.integers(1, k + 1))
                keys = used[at:at + n]
                at += n
                st = h.insert(keys)
                ops.append(0)
                args.append(keys.tolist())
                results.append([])
                statuses.append(st)
            else:
                st, res = h.delete_min()
                ops.append(1)
                args.append([])
                results.append(res.tolist())
                statuses.append(st)
        cases.append({"k": k, "variant": variant, "elide": elide, "max_nodes": max_nodes,
                      "ops": ops, "args": args, "results": results, "statuses": statuses,
                      "counters": h.counters(), "peek": list(h.peek())})
    return cases


def apps_fixture():
    r = O.ref()
    out = {"grid_small": [], "grid_2048": [], "knapsack": []}
    rows = cols = 64
    for src in (0, 1234, 4095):
        d = np.empty(rows * cols, dtype=np.uint64)
        assert r.ref_grid_dijkstra(rows, cols, 1, src, d) == 0
        out["grid_small"].append({"rows": rows, "cols": cols, "seed": 1, "source": src,
                                  "dist": d.tolist()})
    n = 2048 * 2048
    d = np.empty(n, dtype=np.uint64)
    for i in range(8):
        src = i * 524288
        assert r.ref_grid_dijkstra(2048, 2048, 1, src, d) == 0
        out["grid_2048"].append({"source": src, "sum": int(d.sum(dtype=np.uint64)),
                                 "max": int(d.max()),
                                 "unreachable": int((d == np.uint64(2**64 - 1)).sum())})
    for kind in range(4):
        for n_items in (50, 100, 200):
            for rr in (1000, 7000):
                for seed in (1, 2, 3):
                    best = int(r.ref_knapsack_dp(kind, n_items, rr, seed))
                    w = np.empty(n_items, dtype=np.uint32)
                    b = np.empty(n_items, dtype=np.uint32)
                    cap = int(r.ref_generate_knapsack(kind, n_items, rr, seed, w, b))
                    out["knapsack"].append({"type": kind, "n": n_items, "range": rr, "seed": seed,
                                            "capacity": cap, "dp": best,
                                            "w_head": w[:4].tolist(), "b_head": b[:4].tolist()})
    return out


def main():
    with open(os.path.join(OUT, "keygen.json"), "w") as f:
        json.dump(keygen_fixture(), f, indent=1)
    with open(os.path.join(OUT, "heap_histories.json"), "w") as f:
        json.dump(heap_histories(), f)
    with open(os.path.join(OUT, "apps.json"), "w") as f:
        json.dump(apps_fixture(), f)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
