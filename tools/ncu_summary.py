"""Summarise ncu artefacts for profiles/.

    python tools/ncu_summary.py launches <launches.csv>       # per-kernel totals
    python tools/ncu_summary.py full <report.ncu-rep> [key]   # key metrics (+ traffic json key)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warp_latency_issue_stalled_barrier.ratio",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_membar.ratio",
    "smsp__average_warp_latency_issue_stalled_sleeping.ratio",
]


def launches(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    k_name = hdr.index("Kernel Name")
    k_val = hdr.index("Metric Value")
    k_unit = hdr.index("Metric Unit")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[k_val].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
                 "s": 1e3, "second": 1e3}.get(r[k_unit], 1.0)
        name = r[k_name][:90]
        tot[name][0] += 1
        tot[name][1] += v * scale
    total = sum(t for _, t in tot.values())
    out = []
    for name, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        out.append({"kernel": name, "launches": n, "total_ms": round(t, 3),
                    "share": round(t / total, 4) if total else 0})
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def to_bytes(s):
    v, u = s.split()[0].replace(",", ""), s.split()[1] if len(s.split()) > 1 else "byte"
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return float(v) * mul


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        res = full(sys.argv[2])
        print(json.dumps(res, indent=1))
        if len(sys.argv) > 3:
            tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            d = json.load(open(tj)) if os.path.exists(tj) else {}
            r = res[0]
            d[sys.argv[3]] = to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"])
            json.dump(d, open(tj, "w"), indent=1)
