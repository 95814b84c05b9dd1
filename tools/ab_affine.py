"""A/B the affine global kernel on a C2 prefix: in-tree library vs the one in
TA_LIB_PATH_EXPERIMENT (run this script once per library on the same box)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28400_b200 as ta  # noqa: E402

AFF = ta.ScoringScheme(1, -1, -2, -3)
sa, oa = ta.generate("fixed:150:150:150:50000", 0.025, 0.005, 2)
ba = ta.DeviceBatch(sa, oa)
for mode in (0, 1, 2):
    best = 1e9
    for _ in range(4):
        ba.run(AFF, ta.AlignmentMode(mode), ta.EngineConfig(cell_budget=1 << 40))
        best = min(best, ba.stats()["kernel_ms"])
    print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "mode": f"affine-{mode}",
                      "gcups": ba.stats()["cells"] / best / 1e6}), flush=True)
