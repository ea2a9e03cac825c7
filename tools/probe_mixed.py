"""BASELINE config 3 throughput: ins-del pairs on a pre-seeded heap
(proj/src/bench.cpp:60-72,105-113 shape): initial_levels complete levels of
random keys (seed 1 ^ 0x5851f42d4c957f2d), then `pairs` x (insert k keys,
deleteMin) -- 2^26 keys of traffic at the defaults -- in one persistent-
kernel launch, ops interleaved by ticket.  Reports key-ops/s = 2*pairs*k/T
(device time) and, with --ref, the reference's run_workload(InsDelPairs)
on the host cores.  Correctness of this shape is covered by
tests/test_gpu_bulk.py (multiset, invariants, linearizability)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1906_06504_b200 import GeneralizedHeap, Variant, generate_keys, make_ops, phase_ops

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--log2n", type=int, default=26)
ap.add_argument("--levels", type=int, default=14)
ap.add_argument("--variants", default="bu,td")
ap.add_argument("--ref", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="heap debug flags (bh_internal.h kDbg*)")
a = ap.parse_args()
k, n = a.k, 1 << a.log2n
pairs = n // k
seed_nodes = (1 << a.levels) - 1
dev = torch.device("cuda")
seed_keys = generate_keys(seed_nodes * k, 1 ^ 0x5851f42d4c957f2d, key_bits=32)
keys = generate_keys(n, 1, key_bits=32)
kinds = np.tile(np.array([0, 1], np.uint32), pairs)
lens = np.tile(np.array([k, 0], np.uint32), pairs)
offs = np.repeat(np.arange(pairs, dtype=np.uint64) * k, 2)
ops = make_ops(kinds, lens, offs)
d_ops = torch.from_numpy(ops.view(np.uint8)).to(dev)
d_pool = torch.from_numpy(keys.view(np.int32)).to(dev)
d_out = torch.empty(pairs * k, dtype=torch.int32, device=dev)
d_st = torch.zeros(2 * pairs, dtype=torch.int32, device=dev)
d_seed = torch.from_numpy(seed_keys.view(np.int32)).to(dev)
d_seed_ops = torch.from_numpy(phase_ops(0, seed_nodes * k, k).view(np.uint8)).to(dev)
for v in a.variants.split(","):
    for rep in range(a.reps):
        heap = GeneralizedHeap(Variant.BU if v == "bu" else Variant.TD, k, seed_nodes + pairs + 1024, key_bits=32,
                               debug_flags=a.flags)
        s = torch.cuda.current_stream()
        heap.run_ops_ptr(d_seed_ops.data_ptr(), seed_nodes, d_seed.data_ptr(), 0, d_st.data_ptr(), 0, 0,
                         stream=s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        heap.run_ops_ptr(d_ops.data_ptr(), 2 * pairs, d_pool.data_ptr(), d_out.data_ptr(), d_st.data_ptr(), 0, 0,
                         stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ok = bool((d_st == 0).all())
        pk = heap.peek_stats()
        rep_ = heap.check_invariants()
        print(f"mixed ins-del pairs {v} k={k} 2^{a.log2n} keys, {a.levels} seeded levels: {ms:.2f} ms "
              f"key-ops/s {2 * pairs * k / (ms / 1e3):.3e} status_ok={ok} nodes_after={pk.node_count} "
              f"(expect {seed_nodes}) invariants={rep_.ok}", flush=True)
        heap.close()
if a.ref:
    from oracle import oracle as O
    out = np.zeros(7, np.float64)
    w = os.cpu_count()
    for v in a.variants.split(","):
        st = O.ref().ref_run_workload(1 if v == "bu" else 0, k, w, n, 0, 1, a.levels, 100, 1, out)
        print(f"reference run_workload InsDelPairs {v} workers={w}: {out[0]:.3f} s "
              f"key-ops/s {2 * n / out[0]:.3e} (status {st})", flush=True)
