#!/usr/bin/env python3
"""Benchmark: batched insert-all then deleteMin-all on the B200 heap.

BASELINE.json metric: heap key-ops/s for insert+deleteMin at K=1024 on the
configs[1] workload (2^26 random uint32 keys from generate_keys(Random, 2^26,
seed=1), proj/src/workload.cpp:162-180), plus the fraction of the HBM
roofline, with the reference's CPU path timed beside it.

One step = one insert phase (2^26/K insert ops, one persistent-kernel launch)
+ one deleteMin phase (2^26/K delete ops, one launch) on a heap that starts
and ends empty.  key-ops/s = 2N / (T_insert + T_delete), every insert and
every delete of one key counted once.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--k 1024] [--log2n 26]
                    [--variant bu|td] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): independent heap replicas, one per
rank, each running the full workload ("scaling": "weak"); NCCL only carries
the timing barrier/max -- the heap has no data-path collective (SURVEY.md
section 8e).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "heap key-ops/s (insert+deleteMin, K=1024)"
UNIT = "key-ops/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--log2n", type=int, default=26)
    ap.add_argument("--variant", choices=["bu", "td"], default="bu")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ctas", type=int, default=0, help="persistent CTAs (0 = all co-resident)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the u64 line and the profiled root-service run (outside the timed region)")
    return ap.parse_args()


# ------------------------------------------------------------- roofline --
def algorithmic_bytes(n_keys: int, k: int, key_size: int):
    """SURVEY.md section 8(d) walk model, no credit for early stop, elision or
    L2 reuse: an insert of rank r moves K*s*(2 + 2*depth(r)) bytes (input
    read, read+write per interior path node, target write); a delete at m
    resident nodes moves K*s*(4 + 4*depth(m-1)) (root read, result write,
    last-node read, final write, 2 child reads + 2 writes per level), and
    K*s*2 for the last node."""
    n_nodes = (n_keys + k - 1) // k
    ins = dele = 0
    for r in range(1, n_nodes + 1):
        ins += 2 + 2 * (r.bit_length() - 1)
    for m in range(1, n_nodes + 1):
        dele += 2 if m == 1 else 4 + 4 * ((m - 1).bit_length() - 1)
    return ins * k * key_size, dele * k * key_size


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(k: int, log2n: int, variant: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the
    dominant kernel, from the committed ncu --set full summary (or None)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{variant}_k{k}_n{log2n}_delete")
    except Exception:
        return None


def stats(xs):
    return {"min": min(xs), "median": statistics.median(xs), "max": max(xs), "n": len(xs)}


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------- reference ---
def cpu_reference(log2n: int, k: int, variant: str, threads: int, verify: bool = False):
    """The reference's own CPU GeneralizedHeap (oracle/_ref, compiled from
    /root/reference/proj/src), phase-split timer; returns (ins_s, del_s)."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("reference library oracle/_ref/libbatchheap_ref.so not built")
    return O.ref_phase(1 if variant == "bu" else 0, k, 1 << log2n, threads, 1, verify)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(a, rank: int, world: int):
    if rank != 0:
        return
    threads = host_threads()
    # bounded sample: the full configs[1] workload when it fits in a few
    # seconds per step on this host, else 2^24 keys (same K, same generator)
    log2n = a.log2n
    probe = min(20, log2n)
    t_probe = sum(cpu_reference(probe, a.k, a.variant, threads))
    projected = t_probe * (1 << (log2n - probe)) * 1.4
    if projected * (a.steps + a.warmup) > 240:
        log2n = min(log2n, 24)
    n = 1 << log2n
    times = []
    for i in range(a.warmup + a.steps):
        ti, td = cpu_reference(log2n, a.k, a.variant, threads)
        if i >= a.warmup:
            times.append(ti + td)
    t = statistics.mean(times)
    value = 2 * n / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 (reference Key)", "data": "synthetic",
        "config": {"workload": f"insert-then-deleteMin 2^{log2n} random keys (generate_keys seed 1), "
                               f"K={a.k}, {a.variant.upper()} variant, CPU threads={threads}",
                   "k": a.k, "log2n": log2n, "variant": a.variant},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"2^{log2n} keys, K={a.k}, {a.variant.upper()}, {threads} threads, "
                                   f"phase-split timer (oracle/ref_harness.cpp ref_phase)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- extras ----
def root_service(a, dev, keys, stream, flush, value):
    """The root-serial bound: every op holds the root (or
    its delete server's turn) for t_root, so no schedule beats
    N / ((N/K) * (t_root_ins + t_root_del)) round-trip keys/s, i.e. twice
    that in key-ops/s.  t_root from one BH_FLAG_PROFILE step outside the
    timed region (profiling adds its own cycles: an upper estimate of
    t_root, so the fraction below is a lower estimate)."""
    import numpy as np
    import torch
    from paper_1906_06504_b200 import GeneralizedHeap, Variant, phase_ops
    k, n = a.k, 1 << a.log2n
    n_ops = (n + k - 1) // k
    heap = GeneralizedHeap(Variant.BU if a.variant == "bu" else Variant.TD, k, n_ops + 1024, key_bits=32,
                           profile=True, device=dev.index or 0)
    pool = torch.from_numpy(keys.view(np.int32)).to(dev)
    ops_i = torch.from_numpy(phase_ops(0, n, k).view(np.uint8)).to(dev)
    ops_d = torch.from_numpy(phase_ops(1, n, k).view(np.uint8)).to(dev)
    out = torch.empty(n_ops * k, dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        flush.fill_(4)
    stream.synchronize()
    heap.run_ops_ptr(ops_i.data_ptr(), n_ops, pool.data_ptr(), 0, 0, 0, 0, ctas=a.ctas, stream=stream.cuda_stream)
    stream.synchronize()
    p_ins = heap.profile(reset=True)
    heap.run_ops_ptr(ops_d.data_ptr(), n_ops, 0, out.data_ptr(), 0, 0, 0, ctas=a.ctas, stream=stream.cuda_stream)
    stream.synchronize()
    p = heap.profile(reset=True)
    heap.close()
    ghz = 1.965  # B200 SM clock under load (the clocks sampled above)
    us = lambda c, m: c / max(m, 1) / (ghz * 1e3)
    t_ins = us(p_ins["ins_root_hold"], p_ins["ins_ops"])
    # served ops: the server's own (counted in del_ops, one per hold) and
    # the waiters it served (del_served); the rest held the root themselves
    served = p["del_served"] + p["del_serve_holds"]
    unserved = max(p["del_ops"] - p["del_serve_holds"], 0)
    sv = sum(p[f] for f in ("sv_split", "sv_r1", "sv_r2", "sv_r3", "sv_next"))
    t_del_served = us(sv, served)
    t_del_plain = us(p["del_root_hold"], unserved)
    t_del = (served * t_del_served + unserved * t_del_plain) / max(served + unserved, 1)
    bound = 2 * n / (n_ops * (t_ins + t_del) * 1e-6)
    return {"t_root_insert_us": t_ins, "t_root_delete_us": t_del,
            "t_serve_per_delete_us": t_del_served, "t_root_hold_unserved_delete_us": t_del_plain,
            "deletes_served": served, "deletes_unserved": unserved,
            "bound_key_ops_per_s": bound, "achieved_frac_of_bound": value / bound,
            "source": "one BH_FLAG_PROFILE step outside the timed region: mean root hold per insert "
                      "(combining holds included) + per-op delete-server service time"}


def u64_line(a, dev, world):
    """The same step at the reference's own key width (u64, batch.hpp:17)."""
    import numpy as np
    import torch
    from paper_1906_06504_b200 import GeneralizedHeap, Variant, generate_keys, phase_ops
    k, n = a.k, 1 << a.log2n
    n_ops = (n + k - 1) // k
    keys = generate_keys(n, 1, key_bits=64)
    pool = torch.from_numpy(keys.view(np.int64)).to(dev)
    ops_i = torch.from_numpy(phase_ops(0, n, k).view(np.uint8)).to(dev)
    ops_d = torch.from_numpy(phase_ops(1, n, k).view(np.uint8)).to(dev)
    out = torch.empty(n_ops * k, dtype=torch.int64, device=dev)
    seq = torch.empty(n_ops, dtype=torch.int64, device=dev)
    heap = GeneralizedHeap(Variant.BU if a.variant == "bu" else Variant.TD, k, n_ops + 1024, key_bits=64,
                           device=dev.index or 0)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = []
    for i in range(2 + max(2, a.steps // 2)):
        with torch.cuda.stream(stream):
            flush.fill_(5)
        stream.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        heap.run_ops_ptr(ops_i.data_ptr(), n_ops, pool.data_ptr(), 0, 0, 0, 0, ctas=a.ctas, stream=stream.cuda_stream)
        heap.run_ops_ptr(ops_d.data_ptr(), n_ops, 0, out.data_ptr(), 0, 0, seq.data_ptr(), ctas=a.ctas,
                         stream=stream.cuda_stream)
        ev[1].record(stream)
        stream.synchronize()
        if i >= 2:
            times.append(ev[0].elapsed_time(ev[1]))
    drained = out.view(n_ops, k)[torch.argsort(seq)].reshape(-1)[:n]
    ok = bool(torch.equal(drained, torch.sort(pool).values))  # keys < 2^63: signed order == unsigned
    heap.close()
    ms = statistics.mean(times)
    return {"value": world * 2 * n / (ms / 1e3), "unit": UNIT, "dtype": "u64", "ms_per_step": ms,
            "ms_per_step_stats": stats(times), "checked_sorted": ok,
            "workload": f"as config, generate_keys(2^{a.log2n}, seed 1) as uint64 keys"}


# ------------------------------------------------------------------ ours --
def run_ours(a, rank: int, world: int, dist):
    import numpy as np
    import torch

    from paper_1906_06504_b200 import GeneralizedHeap, Variant, generate_keys, phase_ops

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    k, n = a.k, 1 << a.log2n
    n_ops = (n + k - 1) // k
    variant = Variant.BU if a.variant == "bu" else Variant.TD

    keys = generate_keys(n, 1, key_bits=32)  # generate_keys(Random, 2^26, seed=1)
    pool = torch.from_numpy(keys.view(np.int32)).to(dev)
    ops_ins_h = phase_ops(0, n, k)
    ops_del_h = phase_ops(1, n, k)
    ops_ins = torch.from_numpy(ops_ins_h.view(np.uint8)).to(dev)
    ops_del = torch.from_numpy(ops_del_h.view(np.uint8)).to(dev)
    out = torch.empty(n_ops * k, dtype=torch.int32, device=dev)
    seq = torch.empty(n_ops, dtype=torch.int64, device=dev)
    heap = GeneralizedHeap(variant, k, n_ops + 1024, key_bits=32, device=local)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    # L2 flush buffer (> 126 MB L2): written between timed steps, outside them
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        heap.run_ops_ptr(ops_ins.data_ptr(), n_ops, pool.data_ptr(), 0, 0, 0, 0, ctas=a.ctas, stream=sp)
        if ev:
            ev[1].record(stream)
        heap.run_ops_ptr(ops_del.data_ptr(), n_ops, 0, out.data_ptr(), 0, 0, seq.data_ptr(), ctas=a.ctas,
                         stream=sp)
        if ev:
            ev[2].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(a.warmup):
            step()
            flush.fill_(1)
        stream.synchronize()

    # correctness gate on the warm state: the last drain is the sorted input
    order = torch.argsort(seq)
    drained = out.view(n_ops, k)[order].reshape(-1)[:n]
    ref_sorted = torch.sort(pool.to(torch.int64) & 0xFFFFFFFF).values
    ok = bool(torch.equal(drained.to(torch.int64) & 0xFFFFFFFF, ref_sorted))
    if not ok:
        raise SystemExit("bench: drain != sorted(input) -- refusing to report")

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    t_ins, t_del, t_step = [], [], []
    for _ in range(a.steps):
        with torch.cuda.stream(stream):
            flush.fill_(2)
        stream.synchronize()
        if dist:
            dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        step(ev)
        stream.synchronize()
        torch.cuda.synchronize()
        ti, td = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        t_ins.append(ti)
        t_del.append(td)
        t_step.append(ti + td)

    ms = statistics.mean(t_step)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * 2 * n / (ms / 1e3)

    # ---- e2e through the C ABI with pinned HOST buffers (bh_run_ops) ----
    e2e = None
    if not a.no_e2e:
        h_keys = torch.from_numpy(keys.view(np.int32)).pin_memory()
        h_ops_i = torch.from_numpy(ops_ins_h.view(np.uint8)).pin_memory()
        h_ops_d = torch.from_numpy(ops_del_h.view(np.uint8)).pin_memory()
        h_out = torch.empty(n_ops * k, dtype=torch.int32).pin_memory()
        h_seq = torch.empty(n_ops, dtype=torch.int64).pin_memory()
        e2e_times = []
        for i in range(2 + a.steps):
            flush.fill_(3)  # L2 flushed between e2e steps too (outside the timed region)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            heap.run_ops_host_ptr(h_ops_i.data_ptr(), n_ops, h_keys.data_ptr(), n, 0, 0, ctas=a.ctas)
            heap.run_ops_host_ptr(h_ops_d.data_ptr(), n_ops, 0, 0, h_out.data_ptr(), n_ops * k,
                                  seq_ptr=h_seq.data_ptr(), ctas=a.ctas)
            t1 = time.perf_counter()
            if i >= 2:
                e2e_times.append(t1 - t0)
        te = statistics.mean(e2e_times)
        if dist:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        # the e2e result is checked too: the last drain, in sequence order,
        # is the sorted input
        e_out = h_out.to(dev).view(n_ops, k)[torch.argsort(h_seq.to(dev))].reshape(-1)[:n]
        if not torch.equal(e_out.to(torch.int64) & 0xFFFFFFFF, ref_sorted):
            raise SystemExit("bench: e2e drain != sorted(input) -- refusing to report")
        h2d = n * 4 + 2 * n_ops * 16
        d2h = n_ops * k * 4 + n_ops * 8
        e2e = {"value": world * 2 * n / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": te * 1e3,
               "ms_per_step_stats": stats([x * 1e3 for x in e2e_times]),
               "value_stats": stats([world * 2 * n / x for x in e2e_times]),
               "path": "bh_run_ops (C ABI) x2, pinned host buffers, copies + kernels + sync",
               "checked": "last drain == sorted(input)"}
    # clocks sampled over both arms (device-timed steps and e2e steps)
    clocks = sampler.stop() if sampler else None

    if rank != 0:
        return
    ins_b, del_b = algorithmic_bytes(n, k, 4)
    peak, peak_src = measured_peaks()
    td_mean = statistics.mean(t_del) / 1e3
    ti_mean = statistics.mean(t_ins) / 1e3
    achieved = del_b / td_mean / 1e9
    step_s = ms / 1e3
    roofline = {"bound": "hbm", "kernel": "heap_ops_kernel (deleteMin phase launch)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(k, a.log2n, a.variant),
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": del_b,
                "insert_launch": {"achieved": ins_b / ti_mean / 1e9, "algorithmic_bytes": ins_b,
                                  "frac": ins_b / ti_mean / 1e9 / peak},
                "whole_step": {"achieved": (ins_b + del_b) / step_s / 1e9, "algorithmic_bytes": ins_b + del_b,
                               "frac": (ins_b + del_b) / step_s / 1e9 / peak},
                "walk_model": "SURVEY.md 8(d): whole-node read/write per level, no early-stop credit"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"insert-then-deleteMin 2^{a.log2n} random uint32 keys "
                               f"(generate_keys seed 1), K={k}, {a.variant.upper()} variant "
                               f"(BASELINE configs[1])",
                   "k": k, "log2n": a.log2n, "variant": a.variant, "ops_per_phase": n_ops,
                   "ctas": a.ctas or heap.max_ctas, "l2": "256 MB buffer written between timed steps",
                   "parallelism": f"replicas x{world}"},
        "insert_ms": statistics.mean(t_ins), "delete_ms": statistics.mean(t_del),
        "ms_per_step_stats": stats(t_step), "insert_ms_stats": stats(t_ins), "delete_ms_stats": stats(t_del),
        "value_stats": stats([world * 2 * n / (x / 1e3) for x in t_step]),
        "rt_keys_per_s": world * n / (ms / 1e3),
        "roofline": roofline, "clocks": clocks, "gpu_launches": 2 * a.steps,
        "correctness": "drain == sorted(input) checked on device before timing",
    }
    if e2e:
        line["e2e"] = e2e
    if not a.no_extras:
        heap.close()
        del out, seq, pool
        torch.cuda.empty_cache()
        line["root_serial_bound"] = root_service(a, dev, keys, stream, flush, value)
        line["u64"] = u64_line(a, dev, world)
    ref_matrix = os.path.join(ROOT, "profiles", "r2", "ref_matrix.json")
    if os.path.exists(ref_matrix):
        line["cpu_baseline_matrix"] = os.path.relpath(ref_matrix, ROOT)
    if not a.no_cpu_baseline and world == 1:
        try:
            threads = host_threads()
            log2n = a.log2n
            t_probe = sum(cpu_reference(20, k, a.variant, threads))
            if t_probe * (1 << (log2n - 20)) * 1.4 > 30:
                log2n = 24
            ti_c, td_c = cpu_reference(log2n, k, a.variant, threads)
            cv = 2 * (1 << log2n) / (ti_c + td_c)
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": f"2^{log2n} keys, K={k}, {a.variant.upper()}, {threads} threads, "
                                              f"reference GeneralizedHeap phase-split timer"}
        except Exception as exc:  # the reference library may be absent
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {exc}"}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1 and a.impl == "ours":
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist_mod.init_process_group("nccl")
        dist = dist_mod
    if a.impl == "reference":
        run_reference_arm(a, rank, world)
    else:
        run_ours(a, rank, world, dist)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
