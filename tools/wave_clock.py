#!/usr/bin/env python3
"""Dev-only: per-step timeline of wave CTA 1 (variant build with
-DTA_WAVE_CLOCK, selected by TA_LIB_PATH_EXPERIMENT), every thread: C5 score
run, then per tile (r, c) the median work per step (after the mbarrier wait
to the arrival), the median step start relative to the CTA's, face re-reads."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_28400_b200 as ta  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
seqs, offs = ta.generate(f"fixed:{L}:{L}:{L}:1", 0.025, 0.005, 5)
b = ta.DeviceBatch(seqs, offs)
for _ in range(2):
    b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
print(json.dumps({"L": L, "kernel_ms": b.stats()["kernel_ms"]}))
buf = np.zeros((4096, 256, 8), dtype=np.uint64)
rc = ta.lib().ta_debug_wave_clock(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
assert rc == 0, rc
x = buf.astype(np.int64)
live = (x[..., 0] > 0) & (x[..., 1] > 0) & (x[..., 2] > 0) & (x[..., 3] > 0)
steps = np.nonzero(live.any(axis=1))[0]
late = steps[len(steps) // 2:]  # second half: the producer CTA has finished
work = np.where(live, x[..., 2] - x[..., 3], 0)
faces = np.where(live, x[..., 1] - x[..., 3], 0)
res = []
for t in range(256):
    m = live[late, t]
    if not m.any():
        continue
    m6 = m & (x[late, t, 6] > 0) & (x[late, t, 7] > 0)
    tk = float(np.median(x[late, t, 6][m6] - x[late, t, 5][m6])) if m6.any() else -1
    pf = float(np.median(x[late, t, 7][m6] - x[late, t, 6][m6])) if m6.any() else -1
    res.append((float(np.median(work[late, t][m])), t, float(np.median(faces[late, t][m])), float(x[late, t, 4][m].mean()), tk, pf))
res.sort(reverse=True)
per = np.diff(x[late, 0, 0])
print(json.dumps({"late_steps": len(late), "period_us": round(float(np.median(per)) / 1e3, 3)}))
for w, t, f, rr, tk, pf in res[:40]:
    print(json.dumps({"tile": [t // 16, t % 16], "work_us": round(w / 1e3, 3), "to_faces_us": round(f / 1e3, 3),
                      "cpdone_to_taken_us": round(tk / 1e3, 3), "prefetch_issue_us": round(pf / 1e3, 3), "rereads": round(rr, 2)}))
