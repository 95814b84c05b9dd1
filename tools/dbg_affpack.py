import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import ctypes
seqs_offs = None
def run(libpath):
    os.environ["TA_LIB_PATH_EXPERIMENT"] = libpath
    import importlib
    import paper_2605_28400_b200 as ta
    importlib.reload(ta)
    seqs, offs = ta.generate("uniform:64:512:5000", 0.08, 0.01, 4)
    b = ta.DeviceBatch(seqs, offs)
    b.run(ta.ScoringScheme(1, -1, -2, -3), ta.AlignmentMode(0))
    o = b.fetch()
    return o["score"].copy(), np.diff(offs).reshape(-1, 3)
import subprocess, json
res = {}
for v in ("base", "affpack"):
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys, json
sys.path.insert(0, os.getcwd())
os.environ['TA_LIB_PATH_EXPERIMENT'] = 'exp/{v}/libtrioalign_b200.so'
import numpy as np
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate('uniform:64:512:5000', 0.08, 0.01, 4)
b = ta.DeviceBatch(seqs, offs)
b.run(ta.ScoringScheme(1, -1, -2, -3), ta.AlignmentMode(0))
print(json.dumps(b.fetch()['score'].tolist()))
"""], capture_output=True, text=True)
    res[v] = np.array(json.loads(out.stdout.strip().splitlines()[-1]))
import paper_2605_28400_b200 as ta
seqs, offs = ta.generate("uniform:64:512:5000", 0.08, 0.01, 4)
L = np.diff(offs).reshape(-1, 3)
bad = np.flatnonzero(res["base"] != res["affpack"])
print(len(bad), bad[:10].tolist())
for x in bad[:10]: print(x, L[x].tolist(), res["base"][x], res["affpack"][x])
