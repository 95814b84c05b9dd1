#!/usr/bin/env python3
"""Profiling driver: one warm run + one run of the wavefront kernel on a prefix
of the C2 workload (or a given spec), for ncu.  Usage:
  ncu --set full -k regex:wavefront -s 1 -c 1 -o prof python tools/prof_run.py --triplets 20000
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--spec", default="fixed:150:150:150:{n}")
ap.add_argument("--rates", default="0.025:0.005")
ap.add_argument("--seed", type=int, default=2)
ap.add_argument("--triplets", type=int, default=20000)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--rows", action="store_true")
ap.add_argument("--runs", type=int, default=2)
a = ap.parse_args()
mut, ind = (float(x) for x in a.rates.split(":"))
seqs, offs = ta.generate(a.spec.format(n=a.triplets), mut, ind, a.seed)
sch = ta.ScoringScheme(1, -1, -2)
if a.rows:
    for _ in range(a.runs):
        out = ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(a.mode), with_rows=True, cell_budget=1 << 40)
else:
    b = ta.DeviceBatch(seqs, offs)
    for _ in range(a.runs):
        b.run(sch, ta.AlignmentMode(a.mode))
    out = b.fetch()
    print(b.stats())
print("failed", int((out["status"] != 0).sum()))
