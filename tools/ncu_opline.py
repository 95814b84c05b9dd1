#!/usr/bin/env python3
"""Which CUDA source lines execute a given SASS opcode (ncu source page).
usage: ncu_opline.py REPORT OPCODE [top]"""
import collections
import csv
import subprocess
import sys

rep, opc = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cnt = collections.Counter()
src = {}
line = None
fname = ""
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        line = (fname, r[0])
        src[line] = r[1][:100]
        continue
    txt = r[3].strip()
    if txt.startswith("@"):
        txt = txt.split(None, 1)[1]
    if txt.split()[0].rstrip(";") == opc:
        try:
            cnt[line] += int(r[7])
        except ValueError:
            pass
tot = sum(cnt.values())
for ln, n in cnt.most_common(top):
    print(f"{ln[0]}:{ln[1]:>5} {n:.3e} {n / max(tot, 1) * 100:5.1f}%  {src.get(ln, '')}")
