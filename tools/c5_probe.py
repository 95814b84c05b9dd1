#!/usr/bin/env python3
"""C5 score path: one long triplet (1000 / 1500 / 2000 bp) on a resident batch,
best-of-3 kernel time per mode (wave mode), score/end checksum.  usage: c5_probe.py [gap_open]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

OPEN = int(sys.argv[1]) if len(sys.argv) > 1 else 0
tag = os.environ.get("TA_WAVE_DELAY", "default")
for L in (1000, 1500, 2000):
    seqs, offs = ta.generate(f"fixed:{L}:{L}:{L}:1", 0.025, 0.005, 5)
    cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
    b = ta.DeviceBatch(seqs, offs)
    for mode in (0, 1, 2):
        best = 1e9
        for _ in range(3):
            b.run(ta.ScoringScheme(1, -1, -2, OPEN), ta.AlignmentMode(mode), ta.EngineConfig(cell_budget=1 << 40))
            best = min(best, b.stats()["kernel_ms"])
        out = b.fetch()
        print(json.dumps({"delay": tag, "L": L, "open": OPEN, "mode": mode, "ms": round(best, 3),
                          "gcups": round(cells / best / 1e6, 1), "score": int(out["score"][0]),
                          "end": [int(v) for v in out["end"][0]]}), flush=True)
