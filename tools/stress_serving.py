"""Stress of delete serving (tooling): random K, CTA counts, heap sizes and
delete/insert mixes; every run checks results against the sorted input
(phase drains), invariants at quiescence and multiset conservation.

    python tools/stress_serving.py --runs 60 --seed 1
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1906_06504_b200 import GeneralizedHeap, Variant, make_ops, phase_ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=40)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
t0 = time.time()
fails = 0
for run in range(a.runs):
    k = int(rng.choice([256, 512, 1024]))
    # a partial buffer disables serving, so most runs have none
    n = int(rng.integers(1 << 14, 1 << 20)) // k * k + (int(rng.integers(1, k)) if rng.random() < 0.25 else 0)
    probe = GeneralizedHeap(Variant.BU, k, 64, key_bits=32)
    ctas = int(rng.choice([2, 8, 32, probe.max_ctas]))
    probe.close()
    keys = O.generate_keys(n, 1000 + run).astype(np.uint64)
    extra = int(rng.integers(0, 3)) * (n // k // 4) * k
    more = O.generate_keys(max(extra, 1), 5000 + run).astype(np.uint64)[:extra]
    variant = Variant.BU if rng.random() < 0.5 else Variant.TD
    heap = GeneralizedHeap(variant, k, 2 * ((n + extra) // k) + 64, key_bits=32)
    ok = True
    r = heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0, ctas=ctas)
    ok &= bool(np.all(r.status == 0))
    # deletes, with inserts interleaved every `every` ops (0 = none)
    every = int(rng.choice([0, 0, 3, 16]))
    n_del = int(rng.integers(1, (n + extra) // k + 4))
    kinds, lens, offs = [], [], []
    ins_i = 0
    for i in range(n_del):
        kinds.append(1)
        lens.append(0)
        offs.append(i * k)
        if every and (i + 1) % every == 0 and (ins_i + 1) * k <= extra:
            kinds.append(0)
            lens.append(k)
            offs.append(ins_i * k)
            ins_i += 1
    ops = make_ops(np.array(kinds, np.uint32), np.array(lens, np.uint32), np.array(offs, np.uint64))
    pool = more.astype(np.uint32) if extra else np.zeros(1, np.uint32)
    d = heap.run_ops(ops, pool, n_del * k, ctas=ctas)
    ok &= set(np.unique(d.status).tolist()) <= {0, 3}
    rep = heap.check_invariants()
    ok &= rep.ok
    dels = [d.out[o["offset"]:o["offset"] + d.lens[i]] for i, o in enumerate(ops) if o["kind"] == 1]
    inserted = np.concatenate([keys, more[:ins_i * k]])
    got = np.sort(np.concatenate(dels + [heap.collect_resident()]).astype(np.uint64))
    ok &= bool(np.array_equal(got, np.sort(inserted)))
    if not every:  # a pure delete run returns the sorted prefix, op by op in sequence order
        order = np.argsort(d.seq[d.status == 0], kind="stable")
        lens_ok = d.lens[d.status == 0][order]
        outs = d.out.reshape(n_del, k)[d.status == 0][order]
        seq_out = np.concatenate([outs[i, :lens_ok[i]] for i in range(len(order))]).astype(np.uint64) \
            if len(order) else np.zeros(0, np.uint64)
        ok &= bool(np.array_equal(seq_out, np.sort(keys)[:seq_out.size]))
    heap.close()
    fails += not ok
    print(f"run {run:3d} {variant.name} k={k:4d} n={n:8d} extra={extra:7d} ctas={ctas:3d} del={n_del:5d} every={every:2d} "
          f"{'ok' if ok else 'FAIL ' + rep.detail}", flush=True)
print(f"{a.runs - fails}/{a.runs} ok in {time.time() - t0:.1f} s")
sys.exit(1 if fails else 0)
