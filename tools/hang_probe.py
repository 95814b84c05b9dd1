import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
spec, mode, open_ = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
seqs, offs = ta.generate(spec, 0.025, 0.005, 3)
t0 = time.time()
out = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2, open_), ta.AlignmentMode(mode), cfg=ta.EngineConfig(cell_budget=1 << 40))
print(spec, mode, open_, "ok", round(time.time() - t0, 3), int(out["score"][0]), flush=True)
