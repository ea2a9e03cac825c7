"""Diagnostic: insert-all (invariants checked), then delete-all with and
without delete serving, for a few K / variants; reports where results first
go wrong.  Tooling only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle as O
from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops

NO_DEL_SERVE = 0x2000
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << log2n
keys = O.generate_keys(n, 11)
want = O.sort_u64(keys)
FL = [int(x, 0) for x in sys.argv[2:]] or [0, NO_DEL_SERVE]
for k in (1024,):
    for variant in (Variant.BU,):
        for flags in FL:
            heap = GeneralizedHeap(variant, k, n // k + 64, key_bits=32, debug_flags=flags)
            r = heap.run_ops(phase_ops(0, n, k), keys.astype(np.uint32), 0)
            rep = heap.check_invariants()
            res = heap.collect_resident()
            ms_ok = np.array_equal(np.sort(res.astype(np.uint64)), want)
            d = heap.run_ops(phase_ops(1, n, k), np.zeros(0, np.uint32), n)
            out = d.out.reshape(n // k, k)[np.argsort(d.seq, kind="stable")].reshape(-1).astype(np.uint64)
            ok = np.array_equal(out, want)
            bad = -1 if ok else int(np.argmax(out != want))
            srt = bool(np.all(out[:-1] <= out[1:]))
            ms2 = np.array_equal(np.sort(out), want)
            print(f"k={k} {variant.name} flags={flags:#x}: ins_status_ok={bool((r.status==0).all())} inv={rep.ok} "
                  f"resident_multiset={ms_ok} | del_status_ok={bool((d.status==0).all())} drain_ok={ok} sorted={srt} "
                  f"multiset={ms2} first_bad={bad} (batch {bad // k if bad >= 0 else -1})", flush=True)
            heap.close()
