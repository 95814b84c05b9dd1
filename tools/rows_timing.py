import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("fixed:100:100:100:1000", 0.05, 0.0, 1)
for mode in (0, 1, 2):
    for rep in range(4):
        t0 = time.perf_counter()
        ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40)
        print(mode, rep, round(1e3 * (time.perf_counter() - t0), 2), "ms", flush=True)
