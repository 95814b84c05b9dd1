#!/usr/bin/env python3
"""A/B of the traceback (rows) kernels: a C2 prefix through align_arrays
(with_rows), kernel time from the engine stats, best of 3, per mode; one JSON
line per case with a checksum of scores and rows.  TA_LIB_PATH_EXPERIMENT
selects a variant build.  usage: ab_rows.py [--n 20000]"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=20000)
args = ap.parse_args()
seqs, offs = ta.generate(f"fixed:150:150:150:{args.n}", 0.025, 0.005, 2)
cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
lib = os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree")
for mode in (0, 1, 2):
    best = 1e9
    for _ in range(3):
        out = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), with_rows=True,
                              cell_budget=1 << 40)
        best = min(best, ta.last_stats()["kernel_ms"])
    h = hashlib.sha1(out["score"].tobytes() + "".join("".join(r) for r in out["rows"][:2000]).encode()).hexdigest()[:12]
    print(json.dumps({"lib": lib, "case": "C2 rows", "mode": mode, "kernel_gcups": round(cells / best / 1e6, 1),
                      "chk": h}), flush=True)
