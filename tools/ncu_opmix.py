#!/usr/bin/env python3
"""Executed warp-instructions per opcode of an ncu report (SASS source page),
and the issue-cycle estimate of the measured DPX mix model
(profiles/r02_mixpeak.jsonl: half-rate ALU ops 2 cycles, others ~1).
usage: ncu_opmix.py REPORT"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
cnt = collections.Counter()
for r in rows:
    if not r or r[0] in ("Address", "Kernel Name") or len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    try:
        cnt[op.rstrip(";")] += int(r[ix["Instructions Executed"]])
    except ValueError:
        pass
tot = sum(cnt.values())
half = ("VIADDMNMX", "VIMNMX", "IADD3", "PRMT", "ISETP", "SEL", "SHF", "LEA", "VIADD", "IMNMX", "POPC", "FLO", "BREV", "PLOP3")
cyc = 0.0
for op, n in cnt.items():
    base = op.split(".")[0]
    cyc += n * (2.0 if base in half else (0.5 if base == "LOP3" else 1.0))
print(f"total warp-inst {tot:.4e}; model issue-cycles {cyc:.4e}")
for op, n in cnt.most_common(30):
    print(f"  {op:28s} {n:.3e}  {n / tot * 100:5.1f}%")
