"""Aggregate ncu per-SASS stall samples (--page source --csv --print-source
sass) by CUDA source line, using nvdisasm -g line info of the same cubin
(tooling).  usage: ncu_lines.py SASS_CSV DISASM KERNEL_MANGLED [LINE_LO LINE_HI]"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, kern = sys.argv[1], sys.argv[2], sys.argv[3]
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 1 << 30)
# offset -> (file, line)
off2line = {}
cur = None
inside = False
for ln in open(dis):
    if ln.startswith("//---------------------"):
        inside = f".text.{kern} " in ln or ln.rstrip().endswith(f".text.{kern} --------------------------")
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, isamp, inot = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
base = None
agg = defaultdict(lambda: [0, 0])
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    if base is None:
        base = a
    key = off2line.get(a - base, ("?", 0))
    agg[key][0] += int(r[isamp] or 0)
    agg[key][1] += int(r[inot] or 0)
tot = sum(v[0] for v in agg.values())
sel = [(k, v) for k, v in agg.items() if k[0] != "bh_heap.cuh" or lo <= k[1] <= hi]
sel.sort(key=lambda kv: -kv[1][0])
print(f"total samples {tot}")
for (f, l), (s, n) in sel[:45]:
    print(f"{f}:{l:5d}  {s:8d}  {100.0 * s / max(tot, 1):5.1f}%  not-issued {n}")

# stall reasons summed over a region: REGION=file:lo-hi[,file:lo-hi...]
import os
reg = os.environ.get("REGION")
if reg:
    spans = []
    for part in reg.split(","):
        f, rng = part.split(":")
        a, b = rng.split("-")
        spans.append((f, int(a), int(b)))
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = [hdr.index(h) for h in reasons]
    tot_r = defaultdict(int)
    nsel = 0
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        f, l = off2line.get(a - base, ("?", 0))
        if any(f == sf and sa <= l <= sb for sf, sa, sb in spans):
            for h, i in zip(reasons, idx):
                tot_r[h] += int(r[i] or 0)
            nsel += int(r[isamp] or 0)
    print(f"region {reg}: {nsel} samples")
    for h, v in sorted(tot_r.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {h:24s} {v:8d}  {100.0 * v / max(nsel, 1):5.1f}%")
