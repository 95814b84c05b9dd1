#!/usr/bin/env python3
"""Small batches through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): linear score + rows in all modes, a long
(multi-block) and a wave-mode triplet set, affine score + rows, and enough
long triplets to skip wave mode (the 128-wide linear / 64-wide affine block
items)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

rng = np.random.default_rng(3)


def trips(n, lo, hi):
    return [tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=int(L))) for L in rng.integers(lo, hi, size=3))
            for _ in range(n)]


def arrays(ts):
    parts, offs, pos = [], [0], 0
    for t in ts:
        for s in t:
            parts.append(s.encode())
            pos += len(s)
            offs.append(pos)
    return np.frombuffer(b"".join(parts) + b"\0", np.uint8), np.asarray(offs, np.int64)


small = arrays(trips(40, 0, 60))
long_ = arrays(trips(3, 165, 330))
many = [tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=int(L))) for L in (int(rng.integers(0, 4)), b, c))
        for b, c in rng.integers(165, 256, size=(160, 2))]
many = arrays(many)
for mode in (0, 1, 2):
    m = ta.AlignmentMode(mode)
    for sch in (ta.ScoringScheme(1, -1, -2), ta.ScoringScheme(1, -1, -2, -3)):
        for seqs, offs in (small, long_, many):
            ta.align_arrays(seqs, offs, sch, m, cfg=ta.EngineConfig(cell_budget=1 << 40))
        ta.align_arrays(*small, sch, m, with_rows=True, cell_budget=1 << 40)
print("sanitize workload done")
