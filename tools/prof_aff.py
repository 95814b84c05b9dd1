#!/usr/bin/env python3
"""One warm + one profiled affine DeviceBatch run (for ncu).
usage: prof_aff.py SPEC MUT INDEL SEED MODE OPEN"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

spec, mut, indel, seed, mode, op = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
seqs, offs = ta.generate(spec, mut, indel, seed)
b = ta.DeviceBatch(seqs, offs)
cfg = ta.EngineConfig(cell_budget=1 << 40)
for _ in range(2):
    b.run(ta.ScoringScheme(1, -1, -2, op), ta.AlignmentMode(mode), cfg)
    print(spec, mode, b.stats(), flush=True)
