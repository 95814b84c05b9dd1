#!/usr/bin/env python3
"""C5 traceback: one long triplet (1000 / 1500 / 2000 bp) through align_arrays
with rows, every mode (argument: gap_open, default 0); wall and kernel time, GCUPS, a checksum of the rows.
TA_LIB_PATH_EXPERIMENT selects a variant build."""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

lib = os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree")
OPEN = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # gap_open (affine kernels when != 0)
for L in (1000, 1500, 2000):
    seqs, offs = ta.generate(f"fixed:{L}:{L}:{L}:1", 0.025, 0.005, 5)
    cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
    for mode in (0, 1, 2):
        best, kbest = 1e9, 1e9
        for _ in range(2):
            t0 = time.perf_counter()
            out = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2, OPEN), ta.AlignmentMode(mode), with_rows=True,
                                  cell_budget=1 << 40)
            best = min(best, time.perf_counter() - t0)
            kbest = min(kbest, ta.last_stats()["kernel_ms"])
        h = hashlib.sha1(("".join(out["rows"][0]) + str(int(out["score"][0]))).encode()).hexdigest()[:12]
        print(json.dumps({"lib": lib, "case": f"C5 {L} bp rows", "gap_open": OPEN, "mode": mode, "e2e_s": round(best, 4),
                          "kernel_ms": round(kbest, 2), "kernel_gcups": round(cells / kbest / 1e6, 1),
                          "launches": ta.last_stats()["launches"], "chk": h}), flush=True)
