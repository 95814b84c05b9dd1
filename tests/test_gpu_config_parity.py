"""Config-scale parity (BASELINE.md §4 plan): the B200 engine against outputs
of the REFERENCE ITSELF recorded by tests/golden/make_config_parity.py
(reference run_batch over its tiled engine for scores / ends, reference
oracle_align for traceback rows).

  C2  all 1,000,000 triplets in all three modes (and every 64th, semi / local)
  C3  every 64th of 4,000,000 (62,500), all three modes
  C4  every 64th of 100,000 (1,563), all three modes
  C5  1000 / 1500 / 2000 bp single triplets, all three modes (the 2000 bp
      semi-global / local cases have 8.0e9 > 2^32 cells)
  rows: 2,048 C2, 200 C4 and the 1000 bp C5 triplet, all three modes:
      score, end, begin and the three gapped rows

Inputs come from our generator (bit-identical to the reference's: pinned by
tests/golden/gen_hashes.json).  Bar: bit-exact.  With TA_PARITY_OUT set, the
per-config counts are written there as JSON (profiles/r02_parity.json)."""
import gzip
import json
import os
import time

import numpy as np
import pytest

import paper_2605_28400_b200 as ta

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PAR = os.path.join(ROOT, "tests", "golden", "parity")
SCHEME = ta.ScoringScheme(1, -1, -2)
CONFIGS = {
    "C2": ("fixed:150:150:150:1000000", 0.025, 0.005, 2),
    "C3": ("fixed:250:250:250:4000000", 0.025, 0.005, 3),
    "C4": ("uniform:64:512:100000", 0.08, 0.01, 4),
    "C5a": ("fixed:1000:1000:1000:1", 0.025, 0.005, 5),
    "C5b": ("fixed:1500:1500:1500:1", 0.025, 0.005, 5),
    "C5c": ("fixed:2000:2000:2000:1", 0.025, 0.005, 5),
}
MODE_NAMES = {0: "global", 1: "semiglobal", 2: "local"}
RESULTS = []
_DATA = {}

pytestmark = pytest.mark.gpu


def fixture(name):
    path = os.path.join(PAR, name)
    if not os.path.exists(path):
        pytest.fail(f"missing parity fixture {path} (make_config_parity.py)")
    return path


def dataset(name):
    if name not in _DATA:
        _DATA.clear()  # keep one big dataset in host memory at a time
        spec, mut, indel, seed = CONFIGS[name]
        _DATA[name] = ta.generate(spec, mut, indel, seed)
    return _DATA[name]


def subset(seqs, offs, idx):
    lens = np.stack([offs[3 * idx + d + 1] - offs[3 * idx + d] for d in range(3)], axis=1).reshape(-1)
    new_offs = np.zeros(len(lens) + 1, np.int64)
    new_offs[1:] = np.cumsum(lens)
    parts = [seqs[a:b] for a, b in zip(offs[3 * idx], offs[3 * idx + 3])]
    return np.concatenate(parts + [np.zeros(1, np.uint8)]), new_offs


def record(config, mode, kind, n, mism, seconds):
    RESULTS.append({"config": config, "mode": MODE_NAMES[mode], "kind": kind, "compared": int(n),
                    "mismatches": int(mism), "gpu_seconds": round(seconds, 3)})


def compare_scores(config, seqs, offs, mode, want_score, want_end):
    t0 = time.perf_counter()
    out = ta.align_arrays(seqs, offs, SCHEME, ta.AlignmentMode(mode), cfg=ta.EngineConfig(cell_budget=1 << 40))
    dt = time.perf_counter() - t0
    ok = (out["status"] == 0) & (out["score"] == want_score) & (out["end"] == want_end).all(axis=1)
    bad = np.flatnonzero(~ok)
    record(config, mode, "score+end", len(want_score), len(bad), dt)
    assert len(bad) == 0, (config, mode, bad[:10].tolist())


def test_c2_global_all_triplets(gpu_engine):
    seqs, offs = dataset("C2")
    want = np.load(fixture("C2_global.npz"))["score"].astype(np.int32)
    assert len(want) == 1000000
    lens = np.diff(offs).reshape(-1, 3).astype(np.int32)
    compare_scores("C2", seqs, offs, 0, want, lens)


@pytest.mark.parametrize("mode,fname", [(1, "C2_semi.npz"), (2, "C2_local.npz")])
def test_c2_semi_local_all_triplets(gpu_engine, mode, fname):
    """All 1,000,000 C2 triplets in semi-global and local mode (score + end)."""
    if not os.path.exists(os.path.join(PAR, fname)):
        pytest.skip(f"{fname} not generated (make_config_parity.py --only C2_full_modes)")
    z = np.load(fixture(fname))
    want_score, want_end = z["score"].astype(np.int32), z["end"].astype(np.int32)
    assert len(want_score) == 1000000
    seqs, offs = dataset("C2")
    compare_scores("C2", seqs, offs, mode, want_score, want_end)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_strided_samples_all_modes(gpu_engine, name):
    z = np.load(fixture(f"{name}_sample.npz"))
    seqs, offs = dataset(name)
    idx = z["idx"].astype(np.int64)
    s, o = subset(seqs, offs, idx)
    for mode in (0, 1, 2):
        if f"score{mode}" not in z:
            continue
        compare_scores(name, s, o, mode, z[f"score{mode}"], z[f"end{mode}"])


@pytest.mark.parametrize("name", ["C5a", "C5b", "C5c"])
def test_c5_long_triplets_all_modes(gpu_engine, name):
    z = np.load(fixture("C5.npz"))
    seqs, offs = dataset(name)
    for mode in (0, 1, 2):
        compare_scores(name, seqs, offs, mode, z[f"{name}_score{mode}"], z[f"{name}_end{mode}"])


@pytest.mark.parametrize("name", ["C2", "C4", "C5a"])
def test_traceback_rows_vs_reference_oracle(gpu_engine, name):
    with gzip.open(fixture(f"rows_{name}.json.gz"), "rt") as f:
        fx = json.load(f)
    seqs, offs = dataset(name)
    idx = np.asarray(fx["idx"], np.int64)
    s, o = subset(seqs, offs, idx)
    for mode in (0, 1, 2):
        want = fx["modes"][str(mode)]
        t0 = time.perf_counter()
        out = ta.align_arrays(s, o, SCHEME, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40)
        dt = time.perf_counter() - t0
        bad = []
        for x, w in enumerate(want):
            got = (int(out["status"][x]), int(out["score"][x]), out["end"][x].tolist(), out["begin"][x].tolist(),
                   list(out["rows"][x]))
            if got != (0, w["score"], w["end"], w["begin"], w["rows"]):
                bad.append(x)
        record(name, mode, "score+end+begin+rows", len(want), len(bad), dt)
        assert not bad, (name, mode, bad[:10])


def test_write_parity_report():
    """Writes the per-config counts (runs last in this module)."""
    path = os.environ.get("TA_PARITY_OUT")
    if not path:
        pytest.skip("TA_PARITY_OUT not set")
    total = sum(r["compared"] for r in RESULTS)
    with open(path, "w") as f:
        json.dump({"bar": "bit-exact vs the reference (run_batch / oracle_align outputs)",
                   "scheme": [1, -1, -2], "compared_total": total,
                   "mismatches_total": sum(r["mismatches"] for r in RESULTS), "rows": RESULTS}, f, indent=1)
