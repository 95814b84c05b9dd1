#!/usr/bin/env python3
"""Per-source-line profile from an ncu report (--page source, cuda+sass):
every SASS instruction is charged to the CUDA line (file:line) listed above
it; prints the top lines by executed warp-instructions with their stall
samples and the line's top opcodes.  usage: ncu_lines2.py REPORT [top] [opcode]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
only = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
inst = collections.Counter()
samp = collections.Counter()
ops = collections.defaultdict(collections.Counter)
src = {}
fname, cur, ie, ss = "?", None, None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ie, ss = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie:
        continue
    if r[0]:
        cur = f"{fname}:{r[0]}"
        src[cur] = r[1].strip()[:80]
        continue
    if cur is None or not r[3].strip():
        continue
    op = r[3].split()
    op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
    try:
        n, sm = int(r[ie]), int(r[ss])
    except ValueError:
        continue
    if only and not op.startswith(only):
        continue
    inst[cur] += n
    samp[cur] += sm
    ops[cur][op] += n
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp-inst {ti:.4e}  samples {ts}")
for k, v in inst.most_common(top):
    mix = ", ".join(f"{o} {c / v * 100:.0f}%" for o, c in ops[k].most_common(3))
    print(f"{k:22s} {v / ti * 100:5.1f}% inst {samp[k] / ts * 100:5.1f}% stall | {src.get(k, '')[:60]} | {mix}")
