#!/usr/bin/env python3
"""Secondary throughput numbers (one B200): every mode on a C2 prefix
(score path, kernel time from the library's CUDA events), the traceback
(rows) path on C1, mixed-length C4 and single long C5 triplets.
Prints one JSON object per line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

SCH = ta.ScoringScheme(1, -1, -2)


def cells_of(offs):
    return int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())


def score_run(name, spec, rates, seed, mode, reps=2, budget=1 << 40, sch=SCH):
    seqs, offs = ta.generate(spec, *rates, seed)
    b = ta.DeviceBatch(seqs, offs)
    cfg = ta.EngineConfig(cell_budget=budget)
    b.run(sch, ta.AlignmentMode(mode), cfg)
    best = None
    for _ in range(reps):
        b.run(sch, ta.AlignmentMode(mode), cfg)
        st = b.stats()
        best = st["kernel_ms"] if best is None else min(best, st["kernel_ms"])
    out = b.fetch()
    c = cells_of(offs)
    print(json.dumps({"case": name, "mode": ta.mode_name(ta.AlignmentMode(mode)), "gap_open": sch.gap_open,
                      "triplets": len(offs) // 3,
                      "cells": c, "kernel_ms": best, "gcups": c / best / 1e6, "lanes": st["lanes"],
                      "failed": int((out["status"] != 0).sum())}), flush=True)


def rows_run(name, spec, rates, seed, mode):
    seqs, offs = ta.generate(spec, *rates, seed)
    ta.align_arrays(seqs, offs, SCH, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40)
    t0 = time.perf_counter()
    out = ta.align_arrays(seqs, offs, SCH, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40)
    dt = time.perf_counter() - t0
    c = cells_of(offs)
    print(json.dumps({"case": name, "mode": ta.mode_name(ta.AlignmentMode(mode)), "path": "rows (e2e)",
                      "triplets": len(offs) // 3, "cells": c, "seconds": dt, "gcups": c / dt / 1e9,
                      "failed": int((out["status"] != 0).sum())}), flush=True)


AFF = ta.ScoringScheme(1, -1, -2, -3)

if __name__ == "__main__":
    import sys as _sys
    if "--affine" in _sys.argv:
        for mode in (0, 1, 2):
            score_run("C2 prefix 100k affine", "fixed:150:150:150:100000", (0.025, 0.005), 2, mode, sch=AFF)
        score_run("C3 prefix 20k affine", "fixed:250:250:250:20000", (0.025, 0.005), 3, 0, sch=AFF)
        score_run("C4 prefix 5k affine", "uniform:64:512:5000", (0.08, 0.01), 4, 0, sch=AFF)
        _sys.exit(0)
    for mode in (0, 1, 2):
        score_run("C2 prefix 200k", "fixed:150:150:150:200000", (0.025, 0.005), 2, mode)
    for mode in (0, 1, 2):
        rows_run("C1 1000 x 100 bp", "fixed:100:100:100:1000", (0.05, 0.0), 1, mode)
    rows_run("C2 prefix 20k", "fixed:150:150:150:20000", (0.025, 0.005), 2, 0)
    score_run("C3 prefix 100k (250 bp)", "fixed:250:250:250:100000", (0.025, 0.005), 3, 0)
    score_run("C4 prefix 20k (64-512 bp)", "uniform:64:512:20000", (0.08, 0.01), 4, 0)
    for L in (1000, 2000):
        score_run(f"C5 {L} bp", f"fixed:{L}:{L}:{L}:1", (0.025, 0.005), 5, 0, reps=1)
