"""Rows (traceback) path timing: wall time of the public call vs the engine's
own kernel time, per mode, for C1 (1000 x 100 bp) and a C2 prefix.

  python tools/rows_profile.py [--c2 N] [--reps R]
Prints one JSON line per (case, mode)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28400_b200 as ta  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c2", type=int, default=20000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--modes", default="0,1,2")
args = ap.parse_args()

cases = [("C1", "fixed:100:100:100:1000", 0.05, 0.0, 1)]
if args.c2:
    cases.append(("C2", f"fixed:150:150:150:{args.c2}", 0.025, 0.005, 2))
sch = ta.ScoringScheme(1, -1, -2)
for name, spec, mut, ind, seed in cases:
    seqs, offs = ta.generate(spec, mut, ind, seed)
    cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
    for mode in [int(m) for m in args.modes.split(",")]:
        best = 1e9
        for _ in range(args.reps):
            t0 = time.perf_counter()
            out = ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40,
                                  raw_rows=True)
            best = min(best, time.perf_counter() - t0)
        st = ta.last_stats()
        print(json.dumps({"case": name, "mode": mode, "triplets": len(out["score"]), "wall_ms": best * 1e3,
                          "gcups_e2e": cells / best / 1e9, "stats": st,
                          "failed": int((out["status"] != 0).sum())}), flush=True)
