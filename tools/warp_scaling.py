#!/usr/bin/env python3
"""Per-SM throughput vs resident warps: the same kernel family at tile grids
G = 8 / 12 / 16 (2 / 4.5 / 8 warps per SM) on lengths that fill each plane."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

SCH = ta.ScoringScheme(1, -1, -2)
for L, n in ((75, 400000), (115, 300000), (155, 200000)):
    seqs, offs = ta.generate(f"fixed:{L}:{L}:{L}:{n}", 0.0, 0.0, 2)
    b = ta.DeviceBatch(seqs, offs)
    best = 1e9
    for _ in range(3):
        b.run(SCH, ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
        best = min(best, b.stats()["kernel_ms"])
    st = b.stats()
    print(json.dumps({"len": L, "gcups": st["cells"] / best / 1e6, "padded_gcups": st["padded_cells"] / best / 1e6,
                      "lanes": st["lanes"]}), flush=True)
