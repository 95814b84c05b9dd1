import os, sys, json
sys.path.insert(0, os.getcwd())
import paper_2605_28400_b200 as ta
SCH = ta.ScoringScheme(1, -1, -2)
for name, spec, rates, seed in (("C3", "fixed:250:250:250:30000", (0.025, 0.005), 3), ("C4", "uniform:64:512:20000", (0.08, 0.01), 4)):
    s, o = ta.generate(spec, *rates, seed)
    b = ta.DeviceBatch(s, o)
    for mode in (0, 1):
        best = 1e9
        for _ in range(3):
            b.run(SCH, ta.AlignmentMode(mode), ta.EngineConfig(cell_budget=1 << 40))
            best = min(best, b.stats()["kernel_ms"])
        print(json.dumps({"lib": os.environ.get("TA_LIB_PATH_EXPERIMENT", "in-tree"), "cfg": name, "mode": mode, "gcups": b.stats()["cells"] / best / 1e6}), flush=True)
