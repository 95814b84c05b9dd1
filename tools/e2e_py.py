import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("fixed:150:150:150:1000000", 0.025, 0.005, 2)
sch = ta.ScoringScheme(1, -1, -2)
L = ta.lib()
n = (len(offs) - 1) // 3
for rep in range(4):
    t0 = time.perf_counter()
    score = np.zeros(n, np.int32); end = np.zeros((n, 3), np.int32); status = np.zeros(n, np.int32)
    res = ta._Results(ta._ptr(score).value, ta._ptr(end).value, None, ta._ptr(status).value)
    s = sch._c(); opt = ta._options(0, False, None)
    t1 = time.perf_counter()
    rc = L.ta_align_batch(0, ta._ptr(seqs), ta._ptr(offs), n, ctypes.byref(s), ctypes.byref(opt), ctypes.byref(res), None)
    t2 = time.perf_counter()
    r2 = ta.align_arrays(seqs, offs, sch)
    t3 = time.perf_counter()
    print(f"prep {1e3*(t1-t0):.1f} ms  raw call {1e3*(t2-t1):.1f} ms  align_arrays {1e3*(t3-t2):.1f} ms", flush=True)
