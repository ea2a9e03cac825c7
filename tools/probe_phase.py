"""Quick phase-separated timing probe (not the bench): insert-all then
delete-all of n u32 keys at node capacity k, device-resident inputs."""
import argparse
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1906_06504_b200 import GeneralizedHeap, Variant, generate_keys, phase_ops

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=26)
ap.add_argument("--k", type=int, nargs="+", default=[1024])
ap.add_argument("--variant", default="bu")
ap.add_argument("--ctas", type=int, nargs="+", default=[0])
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="heap debug flags (bh_internal.h kDbg*)")
a = ap.parse_args()
n = 1 << a.log2n
dev = torch.device("cuda")
keys = generate_keys(n, 1, key_bits=32)
pool = torch.from_numpy(keys.view(np.int32)).to(dev)
for k in a.k:
    for ctas in a.ctas:
        for rep in range(a.reps):
            heap = GeneralizedHeap(Variant.BU if a.variant == "bu" else Variant.TD, k, n // k + 1024, key_bits=32, profile=a.profile, debug_flags=a.flags)
            n_ops = n // k
            ops_i = torch.from_numpy(phase_ops(0, n, k).view(np.uint8)).to(dev)
            ops_d = torch.from_numpy(phase_ops(1, n, k).view(np.uint8)).to(dev)
            out = torch.empty(n, dtype=torch.int32, device=dev)
            st = torch.zeros(n_ops, dtype=torch.int32, device=dev)
            seq = torch.empty(n_ops, dtype=torch.int64, device=dev)
            s = torch.cuda.current_stream()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record(s)
            heap.run_ops_ptr(ops_i.data_ptr(), n_ops, pool.data_ptr(), 0, st.data_ptr(), 0, 0, ctas=ctas, stream=s.cuda_stream)
            e1.record(s)
            heap.run_ops_ptr(ops_d.data_ptr(), n_ops, 0, out.data_ptr(), st.data_ptr(), 0, seq.data_ptr(), ctas=ctas, stream=s.cuda_stream)
            e2.record(s)
            torch.cuda.synchronize()
            ti, td = e0.elapsed_time(e1), e1.elapsed_time(e2)
            order = torch.argsort(seq)
            stream = out.view(n_ops, k)[order].reshape(-1)
            ok = bool((stream[:-1].to(torch.int64) & 0xFFFFFFFF).le(stream[1:].to(torch.int64) & 0xFFFFFFFF).all())
            c = heap.counters()
            print(f"k={k} ctas={ctas or heap.max_ctas} n=2^{a.log2n} {a.variant}: insert {ti:.2f} ms "
                  f"delete {td:.2f} ms  key-ops/s {2*n/((ti+td)/1e3):.3e} sorted={ok} "
                  f"merges={c.merges} elided={c.elided_merges} early={c.early_stops} visits={c.propagation_node_visits}",
                  flush=True)
            if a.profile:
                p = heap.profile(reset=False)
                ghz = 1.9
                def us(c, ops):
                    return c / max(ops, 1) / (ghz * 1e3)
                print(f"   ins/op us: sort {us(p['ins_sort'], p['ins_ops']):.2f} rootwait {us(p['ins_root_wait'], p['ins_ops']):.2f} "
                      f"roothold {us(p['ins_root_hold'], p['ins_ops']):.2f} rest {us(p['ins_rest'], p['ins_ops']):.2f} | "
                      f"del/op us: rootwait {us(p['del_root_wait'], p['del_ops']):.2f} roothold {us(p['del_root_hold'], p['del_ops']):.2f} "
                      f"heapify {us(p['del_rest'], p['del_ops']):.2f} childwait {us(p['child_wait'], p['del_ops']):.2f} "
                      f"levels/del {p['levels']/max(p['del_ops'],1):.2f}", flush=True)
                d = p['del_ops']; lv = max(p['levels'] - d, 1)
                print(f"   del root step us: head {us(p['rs_head'], d):.2f} child {us(p['rs_child'], d):.2f} last {us(p['rs_last'], d):.2f} "
                      f"load {us(p['rs_load'], d):.2f} fill {us(p['rs_fill'], d):.2f} | per level us: acq {us(p['lv_acq'], lv):.2f} "
                      f"load {us(p['lv_load'], lv):.2f} merge {us(p['lv_merge'], p['levels']):.2f} rel {us(p['lv_rel'], p['levels']):.2f}", flush=True)
                bl = max(p['bu_levels'], 1)
                print(f"   insert combining: served {p['served']} in {p['serve_holds']} holds | climb levels/ins {p['bu_levels']/max(p['ins_ops'],1):.2f} "
                      f"parent-claim us {us(p['bu_parent'], bl):.2f} retake us {us(p['bu_retake'], bl):.2f}", flush=True)
                print(f"   delete root split: refill half {us(p['split_a'], d):.2f} us, children half {us(p['split_b'], d):.2f} us", flush=True)
                sv = max(p['del_served'] + p['del_serve_holds'], 1)
                print(f"   delete serving: served {p['del_served']} in {p['del_serve_holds']} holds | per op us: "
                      f"split {us(p['sv_split'], sv):.2f} (refill {us(p['sv_a'], sv):.2f}; H0+lo0 {us(p['sv_b'], sv):.2f} then claims {us(p['sv_claim'], sv):.2f}) "
                      f"r1 {us(p['sv_r1'], sv):.2f} "
                      f"r2 {us(p['sv_r2'], sv):.2f} r3 {us(p['sv_r3'], sv):.2f} next {us(p['sv_next'], sv):.2f}", flush=True)
                print(f"   insert root holds (claim_and_serve): {p['hold_cs_n']} x {us(p['hold_cs'], p['hold_cs_n']):.2f} us | "
                      f"climb root steps: {p['climb_root_n']} x {us(p['climb_root'], p['climb_root_n']):.2f} us | "
                      f"claim_and_serve: to entry {us(p['cs1'], p['hold_cs_n']):.2f} look-ups {us(p['cs2'], p['hold_cs_n']):.2f} "
                      f"claims {us(p['cs3'], p['hold_cs_n']):.2f} to fence {us(p['cs4'], p['hold_cs_n']):.2f} us", flush=True)
                lvp = heap.profile_levels()
                rows = [f"L{i}:{lvp['steps'][i]}/{lvp['claim_cycles'][i] / (ghz * 1e3):.1f}/{lvp['hold_cycles'][i] / (ghz * 1e3):.2f}"
                         for i in range(32) if lvp['steps'][i]]
                print("   BU climb per parent level (steps / parent-claim us / claim-to-release us): " + " ".join(rows), flush=True)
                s3 = max(p['s3_ops'], 1)
                print(f"   three-level server: {p['s3_ops']} ops | per op us: op {us(p['s3_op'], s3):.2f} r0 {us(p['s3_r0'], s3):.2f} "
                      f"wait-refill {us(p['s3_wait_rf'], s3):.2f} r1 {us(p['s3_r1'], s3):.2f} wait-claim {us(p['s3_wait_c3'], s3):.2f} "
                      f"r2 {us(p['s3_r2'], s3):.2f} r3 {us(p['s3_r3'], s3):.2f} | claim warp {us(p['s3_claim'], s3):.2f} "
                      f"refill warps {us(p['s3_refill'], s3):.2f} control warp {us(p['s3_ctl'], s3):.2f} | "
                      f"between ops: record {us(p['s3_rec'], s3):.2f} wake {us(p['s3_wake'], s3):.2f} "
                      f"post {us(p['s3_post'], s3):.2f} start {us(p['s3_start'], s3):.2f}", flush=True)
            heap.close()
