#!/usr/bin/env python3
"""Quick A/B of the score kernels: every mode on a C2 prefix (and optionally a
C4 prefix), kernel time from the engine's CUDA events, best of 3; prints one
JSON line per case with a result checksum.  TA_LIB_PATH_EXPERIMENT selects a
variant build of the same ABI.
usage: ab_quick.py [--n 200000] [--c4 0] [--c3 0] [--modes 0,1,2] [--gap-open 0]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--c4", type=int, default=0)
ap.add_argument("--c3", type=int, default=0)
ap.add_argument("--modes", default="0,1,2")
ap.add_argument("--gap-open", type=int, default=0)
args = ap.parse_args()
sch = ta.ScoringScheme(1, -1, -2, args.gap_open)
cases = [("C2", f"fixed:150:150:150:{args.n}", 0.025, 0.005, 2)]
if args.c4:
    cases.append(("C4", f"uniform:64:512:{args.c4}", 0.08, 0.01, 4))
if args.c3:
    cases.append(("C3", f"fixed:250:250:250:{args.c3}", 0.025, 0.005, 3))
lib = os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree")
for name, spec, mut, ind, seed in cases:
    seqs, offs = ta.generate(spec, mut, ind, seed)
    cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
    b = ta.DeviceBatch(seqs, offs)
    for mode in [int(m) for m in args.modes.split(",")]:
        cfg = ta.EngineConfig(cell_budget=1 << 40)
        best = 1e9
        for _ in range(3):
            b.run(sch, ta.AlignmentMode(mode), cfg)
            best = min(best, b.stats()["kernel_ms"])
        out = b.fetch()
        chk = int((out["score"].astype(np.int64) * 131 + out["end"].astype(np.int64).sum(axis=1)).sum())
        print(json.dumps({"lib": lib, "case": name, "mode": mode, "gap_open": args.gap_open,
                          "gcups": round(cells / best / 1e6, 1), "chk": chk,
                          "failed": int((out["status"] != 0).sum())}), flush=True)
