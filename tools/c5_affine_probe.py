#!/usr/bin/env python3
"""Config C5 (single long triplet) through the affine kernels: kernel time."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

for L in (1000, 2000):
    seqs, offs = ta.generate(f"fixed:{L}:{L}:{L}:1", 0.025, 0.005, 5)
    b = ta.DeviceBatch(seqs, offs)
    sch = ta.ScoringScheme(1, -1, -2, -3)
    b.run(sch, ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
    b.run(sch, ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
    st = b.stats()
    print(json.dumps({"case": f"C5 {L} bp affine", "kernel_ms": st["kernel_ms"], "gcups": st["cells"] / st["kernel_ms"] / 1e6,
                      "score": int(b.fetch()["score"][0])}), flush=True)
