#!/usr/bin/env python3
"""Aggregate an ncu source page (cuda,sass) by CUDA source line:
instructions executed and stall samples.  usage: ncu_lines.py REPORT [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = []
cur = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row (aggregate of its SASS)
        try:
            agg.append((int(r[7]), int(r[4]), r[0], r[1][:90]))
        except ValueError:
            pass
tot_i = sum(a[0] for a in agg)
tot_s = sum(a[1] for a in agg)
print(f"total inst {tot_i:.3e}  samples {tot_s}")
for inst, samp, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{ln:>5} {inst / tot_i * 100:5.1f}% inst {samp / max(tot_s, 1) * 100:5.1f}% stall  {src}")
