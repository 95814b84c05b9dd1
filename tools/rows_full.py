"""Traceback (rows) path at the full C2 size: 1M x 150 bp through the public
call (align_arrays with raw row planes: host ASCII in, host row planes out),
per mode, after one full-size warm-up call (buffer growth).  Prints one JSON line per mode."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28400_b200 as ta  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
modes = [int(m) for m in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2").split(",")]
seqs, offs = ta.generate(f"fixed:150:150:150:{n}", 0.025, 0.005, 2)
cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
sch = ta.ScoringScheme(1, -1, -2)
# warm-up at full size: the first call grows the engine's device / pinned buffers
ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(0), with_rows=True, cell_budget=1 << 40, raw_rows=True)
for mode in modes:
    t0 = time.perf_counter()
    out = ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40, raw_rows=True)
    dt = time.perf_counter() - t0
    st = ta.last_stats()
    print(json.dumps({"case": f"C2 fixed:150:150:150:{n}", "mode": mode, "e2e_s": dt, "e2e_gcups": cells / dt / 1e9,
                      "kernel_ms": st["kernel_ms"], "kernel_gcups": cells / st["kernel_ms"] / 1e6,
                      "dir_bytes": st["dir_bytes"], "rows_bytes": int(out["row_len"].astype(np.int64).sum()) * 3,
                      "failed": int((out["status"] != 0).sum())}), flush=True)
