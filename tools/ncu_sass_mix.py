#!/usr/bin/env python3
"""Opcode mix and stall samples of one kernel from an ncu report's SASS page.
usage: ncu_sass_mix.py REPORT [top]
Prints instructions executed per opcode (warp-level) and stall samples."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
inst = collections.Counter()
samp = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0] if src else "?"
    try:
        inst[op] += int(r[ie])
        samp[op] += int(r[ss])
    except ValueError:
        pass
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total warp-inst {ti:.4e}  stall samples {ts}")
for op, v in inst.most_common(top):
    print(f"{op:28s} {v / ti * 100:6.2f}% inst  {samp[op] / max(ts, 1) * 100:6.2f}% samples")
