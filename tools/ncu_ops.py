#!/usr/bin/env python3
"""Executed warp-instructions per SASS opcode from an ncu report.
usage: ncu_ops.py REPORT [top]"""
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
ii = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
st = collections.Counter()
for r in rows[2:]:
    if len(r) <= ii:
        continue
    txt = r[1].strip()
    if txt.startswith("@"):
        txt = txt.split(None, 1)[1]
    op = txt.split()[0].rstrip(";") if txt else "?"
    try:
        ops[op] += int(r[ii])
        st[op] += int(r[si])
    except ValueError:
        pass
tot = sum(ops.values())
tots = sum(st.values())
print(f"total warp-inst {tot:.4e}")
for op, n in ops.most_common(top):
    print(f"{op:28s} {n:.3e} {n / tot * 100:5.1f}%  stall {st[op] / tots * 100:5.1f}%")
