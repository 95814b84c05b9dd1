import os, sys
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("fixed:150:150:150:6000", 0.025, 0.005, 2)
for mode in (0, 1):
    ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40, raw_rows=True)
