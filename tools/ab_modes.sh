#!/bin/bash
# A/B: C2 prefix global/local through the in-tree library and an experiment build.
# usage: tools/ab_modes.sh <variant libtrioalign_b200.so>
set -e
cat > /tmp/ab.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
SCH = ta.ScoringScheme(1, -1, -2)
seqs, offs = ta.generate("fixed:150:150:150:200000", 0.025, 0.005, 2)
b = ta.DeviceBatch(seqs, offs)
for mode in (0, 1, 2):
    cfg = ta.EngineConfig(cell_budget=1 << 40)
    best = 1e9
    for _ in range(3):
        b.run(SCH, ta.AlignmentMode(mode), cfg)
        best = min(best, b.stats()["kernel_ms"])
    cells = 674981204837
    print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "mode": mode, "gcups": cells / best / 1e6}))
s3, o3 = ta.generate("fixed:250:250:250:30000", 0.025, 0.005, 3)
b3 = ta.DeviceBatch(s3, o3)
best = 1e9
for _ in range(3):
    b3.run(SCH, ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
    best = min(best, b3.stats()["kernel_ms"])
print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "mode": "C3-global", "gcups": b3.stats()["cells"] / best / 1e6}))
AFF = ta.ScoringScheme(1, -1, -2, -3)
sa, oa = ta.generate("fixed:150:150:150:50000", 0.025, 0.005, 2)
ba = ta.DeviceBatch(sa, oa)
best = 1e9
for _ in range(3):
    ba.run(AFF, ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
    best = min(best, ba.stats()["kernel_ms"])
print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "mode": "affine-global", "gcups": ba.stats()["cells"] / best / 1e6}))
PY
python /tmp/ab.py
TA_LIB_PATH_EXPERIMENT="$1" python /tmp/ab.py
python /tmp/ab.py
TA_LIB_PATH_EXPERIMENT="$1" python /tmp/ab.py
