#!/usr/bin/env python3
"""BASELINE.json configs C3 (4M x 250 bp) and C4 (100k x 64-512 bp) at their
full sizes on one B200: kernel-only GCUPS (device-resident batch, best of 2),
linear and affine (gap_open -3), plus the mode-ordering property on C4."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

CFG = ta.EngineConfig(cell_budget=1 << 40)


def timed(b, sch, mode, reps=2):
    best = None
    for _ in range(reps):
        b.run(sch, ta.AlignmentMode(mode), CFG)
        ms = b.stats()["kernel_ms"]
        best = ms if best is None else min(best, ms)
    return best


for name, spec, rates, seed, modes, affine in (("C3", "fixed:250:250:250:4000000", (0.025, 0.005), 3, (0,), True),
                                                ("C4", "uniform:64:512:100000", (0.08, 0.01), 4, (0, 1, 2), True)):
    t0 = time.perf_counter()
    seqs, offs = ta.generate(spec, *rates, seed)
    gen_s = time.perf_counter() - t0
    b = ta.DeviceBatch(seqs, offs)
    n = (len(offs) - 1) // 3
    scores = {}
    for mode in modes:
        ms = timed(b, ta.ScoringScheme(1, -1, -2), mode, reps=2 if name == "C4" else 1)
        out = b.fetch()
        scores[mode] = out["score"].copy()
        st = b.stats()
        print(json.dumps({"config": name, "spec": spec, "triplets": n, "mode": ta.mode_name(ta.AlignmentMode(mode)),
                          "gap": "linear", "cells": st["cells"], "kernel_ms": ms, "gcups": st["cells"] / ms / 1e6,
                          "failed": int((out["status"] != 0).sum()), "generate_s": round(gen_s, 1)}), flush=True)
    if len(modes) == 3:
        ok = bool((scores[2] >= scores[1]).all() and (scores[1] >= scores[0]).all())
        print(json.dumps({"config": name, "property": "local >= semiglobal >= global on every triplet", "holds": ok}),
              flush=True)
    if affine:
        ms = timed(b, ta.ScoringScheme(1, -1, -2, -3), 0, reps=1)
        st = b.stats()
        out = b.fetch()
        print(json.dumps({"config": name, "mode": "global", "gap": "affine open -3", "cells": st["cells"], "kernel_ms": ms,
                          "gcups": st["cells"] / ms / 1e6, "failed": int((out["status"] != 0).sum())}), flush=True)
    b.close()
