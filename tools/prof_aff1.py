import os, sys
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("fixed:150:150:150:6000", 0.025, 0.005, 2)
b = ta.DeviceBatch(seqs, offs)
b.run(ta.ScoringScheme(1, -1, -2, -3), ta.AlignmentMode(0))
print(b.stats())
