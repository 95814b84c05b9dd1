"""C3 / C4 prefixes (kernel-only GCUPS) for A/B of the narrower block items:
linear 128-wide (TA_T8_COST) and affine 64-wide (TA_AFF4_COST); run once per
setting (100 disables them)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_28400_b200 as ta  # noqa: E402

SCH = ta.ScoringScheme(1, -1, -2)
for name, spec, rates, seed, modes in (("C3", "fixed:250:250:250:100000", (0.025, 0.005), 3, (0,)),
                                       ("C4", "uniform:64:512:100000", (0.08, 0.01), 4, (0, 1, 2))):
    seqs, offs = ta.generate(spec, *rates, seed)
    b = ta.DeviceBatch(seqs, offs)
    for mode in modes:
        best = 1e9
        for _ in range(2):
            b.run(SCH, ta.AlignmentMode(mode), ta.EngineConfig(cell_budget=1 << 40))
            best = min(best, b.stats()["kernel_ms"])
        st = b.stats()
        out = b.fetch()
        print(json.dumps({"t8_cost": os.environ.get("TA_T8_COST", "default"), "config": name, "mode": mode,
                          "gcups": st["cells"] / best / 1e6, "padded_frac": st["cells"] / max(1, st.get("padded_cells", 1)),
                          "score_sum": int(out["score"].sum()), "failed": int((out["status"] != 0).sum())}), flush=True)
    best = 1e9
    for _ in range(2):
        b.run(ta.ScoringScheme(1, -1, -2, -3), ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
        best = min(best, b.stats()["kernel_ms"])
    st = b.stats()
    out = b.fetch()
    print(json.dumps({"aff4_cost": os.environ.get("TA_AFF4_COST", "default"), "config": name, "mode": "affine-0",
                      "gcups": st["cells"] / best / 1e6, "padded_frac": st["cells"] / max(1, st.get("padded_cells", 1)),
                      "score_sum": int(out["score"].sum()), "failed": int((out["status"] != 0).sum())}), flush=True)
    b.close()
