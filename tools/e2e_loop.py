#!/usr/bin/env python3
"""bench.py's e2e leg in isolation: align_arrays on the C2 batch, warm + K timed."""
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2605_28400_b200 as ta  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
seqs, offs = ta.generate(f"fixed:150:150:150:{n}", 0.025, 0.005, 2)
sch = ta.ScoringScheme(1, -1, -2)
for rep in range(4):
    t0 = time.perf_counter()
    ta.align_arrays(seqs, offs, sch)
    print(f"align_arrays {time.perf_counter() - t0:.3f}s", flush=True)
