import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_28400_b200 as ta
from oracle.pyoracle import Oracle
o = Oracle()
seqs, offs = ta.generate("fixed:150:150:150:8", 0.025, 0.005, 2)
out = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(1), cfg=ta.EngineConfig(cell_budget=1 << 40))
trips = ta.triplets_from_arrays(seqs, offs)
for x, t in enumerate(trips):
    w = o.align((t.s0, t.s1, t.s2), (1, -1, -2), 1, with_rows=False)
    print(x, int(out["score"][x]), out["end"][x].tolist(), "want", w["score"], w["end"])
