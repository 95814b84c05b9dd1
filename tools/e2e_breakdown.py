#!/usr/bin/env python3
"""Where does end-to-end time go?  create (H2D + pack) / run (kernels +
host planning) / fetch (D2H) for the C2 batch through the C-ABI."""
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
t0 = time.perf_counter()
seqs, offs = ta.generate(f"fixed:150:150:150:{n}", 0.025, 0.005, 2)
t1 = time.perf_counter()
print(f"generate {t1 - t0:.3f}s  bytes {seqs.nbytes / 1e6:.1f} MB")
sch = ta.ScoringScheme(1, -1, -2)
for rep in range(3):
    t0 = time.perf_counter()
    b = ta.DeviceBatch(seqs, offs)
    t1 = time.perf_counter()
    b.run(sch)
    t2 = time.perf_counter()
    out = b.fetch()
    t3 = time.perf_counter()
    st = b.stats()
    b.close()
    t4 = time.perf_counter()
    print(f"create {t1 - t0:.3f}  run {t2 - t1:.3f} (kernel {st['kernel_ms'] / 1e3:.3f})  fetch {t3 - t2:.3f}  "
          f"destroy {t4 - t3:.3f}")
t0 = time.perf_counter()
r = ta.align_arrays(seqs, offs, sch)
print(f"align_arrays {time.perf_counter() - t0:.3f}s")
