import os, sys
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("fixed:1000:1000:1000:1", 0.025, 0.005, 5)
b = ta.DeviceBatch(seqs, offs)
for _ in range(2):
    b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
print(b.stats())
