#!/usr/bin/env python3
"""Summarise a ptxas -v log: registers / spills per heap_ops_kernel instance
(tooling: run on paper_1906_06504_b200/csrc/_obj*/bh_kernels_u*.o.ptxas.log)."""
import re
import subprocess
import sys

for path in sys.argv[1:]:
    fn = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            fn = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and fn:
            spill = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and fn and "heap_ops_kernel" in fn:
            print(f"{fn[:90]:90s} regs={m.group(1)} spill_st={spill}")
