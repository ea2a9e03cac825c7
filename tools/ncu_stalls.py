"""Warp-stall sampling summary of an ncu --set full report (tooling): the
share of each smsp__pcsamp_warps_issue_stalled_* reason among all samples.
With the source page (reports taken with --import-source on), also the
source lines holding the most samples.
usage: ncu_stalls.py REPORT.ncu-rep [LABEL] > out.json"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
pre = "smsp__pcsamp_warps_issue_stalled_"
st = {h[len(pre):]: float(v.replace(",", "")) for h, v in zip(hdr, vals)
      if h.startswith(pre) and not h.endswith("_not_issued")}
tot = sum(st.values()) or 1.0
out = {"report": label, "samples": int(tot),
       "share": {k: round(v / tot, 4) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v > 0}}
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg, cur = {}, None
for r in csv.reader(io.StringIO(src)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif len(r) > 5 and r[0].isdigit():
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        if v > 0:
            agg[f"{cur}:{r[0]}"] = agg.get(f"{cur}:{r[0]}", 0.0) + v
if agg:
    t = sum(agg.values())
    out["top_lines"] = {k: round(v / t, 4) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]}
json.dump(out, sys.stdout, indent=1)
print()
