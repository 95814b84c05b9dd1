"""C1 rows path (1000 x 100 bp, score + traceback) wall time per mode, best of
10 calls through align_arrays (A/B with TA_LIB_PATH_EXPERIMENT)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28400_b200 as ta  # noqa: E402

seqs, offs = ta.generate("fixed:100:100:100:1000", 0.05, 0.0, 1)
for mode in (0, 1, 2):
    best = 1e9
    for _ in range(10):
        t0 = time.perf_counter()
        ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), with_rows=True,
                        cell_budget=1 << 40)
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "mode": mode, "best_ms": best * 1e3}))
