#!/usr/bin/env python3
"""Stall reasons of an ncu report's SASS page, summed per opcode and over the
whole kernel (all samples), plus the top instructions by long-scoreboard /
any chosen reason.  usage: ncu_stalls.py REPORT [reason] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
focus = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
inst = []
for r in rows:
    if not r or r[0] in ("Address", "Kernel Name") or len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()
    op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
    for h in reasons:
        try:
            v = int(r[ix[h]])
        except ValueError:
            continue
        tot[h] += v
        byop[op.split(".")[0]][h] += v
    try:
        inst.append((int(r[ix[focus]]), r[0][-5:], src[:70]))
    except ValueError:
        pass
T = sum(tot.values()) or 1
print("kernel stall shares:", ", ".join(f"{k[6:]} {v / T * 100:.1f}%" for k, v in tot.most_common(12)))
print(f"\nby opcode (share of all samples), focus {focus}:")
opt = sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:14]
for op, c in opt:
    s = sum(c.values())
    print(f"  {op:12s} {s / T * 100:5.1f}%  " + ", ".join(f"{k[6:]} {v / T * 100:.1f}" for k, v in c.most_common(4)))
print(f"\ntop instructions by {focus}:")
for v, a, s in sorted(inst, reverse=True)[:top]:
    print(f"  {v / T * 100:5.2f}%  {a}  {s}")
