#!/usr/bin/env python3
"""One warm + one profiled DeviceBatch run of a config prefix (for ncu).
usage: prof_one.py SPEC MUT INDEL SEED MODE [reps]"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

spec, mut, indel, seed, mode = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
seqs, offs = ta.generate(spec, mut, indel, seed)
b = ta.DeviceBatch(seqs, offs)
cfg = ta.EngineConfig(cell_budget=1 << 40)
for _ in range(reps):
    b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), cfg)
    print(spec, mode, b.stats(), flush=True)
