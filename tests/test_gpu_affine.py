"""GPU parity of the affine-gap kernels (affine.cuh) through the C-ABI.

The reference has linear gaps only, so (SPEC-AFFINE.md):
* with gap_open = 0 the affine kernels (forced with gap_model = 1) must
  reproduce the reference's own golden vectors - scores, ends and rows;
* with gap_open < 0 they must equal the builder's affine oracle
  (oracle/affine_oracle.c, pinned by tests/test_affine_oracle.py) bit for bit:
  score, end, begin and rows, in every mode, for s16x2 and int32 lanes,
  single-block and multi-block (long) triplets.
Needs a B200."""
import numpy as np
import pytest

import paper_2605_28400_b200 as ta
from conftest import load_golden

pytestmark = pytest.mark.gpu

MODES = (0, 1, 2)


def trips_to_arrays(trips):
    parts, offs, pos = [], [0], 0
    for t in trips:
        for s in t:
            parts.append(s.encode())
            pos += len(s)
            offs.append(pos)
    return np.frombuffer(b"".join(parts) + b"\0", np.uint8), np.asarray(offs, np.int64)


def run(trips, sch, mode, rows=False, force=False):
    seqs, offs = trips_to_arrays(trips)
    cfg = ta.EngineConfig(cell_budget=1 << 40, gap_model=1 if force else 0)
    return ta.align_arrays(seqs, offs, ta.ScoringScheme(*sch), ta.AlignmentMode(mode), cfg=cfg,
                           with_rows=rows, cell_budget=(1 << 40) if rows else None)


def rand_trips(rng, n, lo, hi):
    return [tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=int(L))) for L in rng.integers(lo, hi, size=3))
            for _ in range(n)]


@pytest.mark.parametrize("mode", MODES)
def test_open_zero_reproduces_reference_golden(gpu_engine, mode):
    cases = [c for c in load_golden("small_rows.json.gz") if c["mode"] == mode]
    by_scheme = {}
    for c in cases:
        by_scheme.setdefault(tuple(c["scheme"]), []).append(c)
    for sch, cs in by_scheme.items():
        trips = [c["t"] for c in cs]
        sc = run(trips, sch + (0,), mode, force=True)
        rw = run(trips, sch + (0,), mode, rows=True, force=True)
        for x, c in enumerate(cs):
            want = c["oracle"]
            assert int(sc["status"][x]) == 0 and int(rw["status"][x]) == 0
            assert int(sc["score"][x]) == want["score"] and list(sc["end"][x]) == want["end"], (sch, c["t"])
            assert int(rw["score"][x]) == want["score"] and list(rw["end"][x]) == want["end"], (sch, c["t"])
            assert list(rw["begin"][x]) == want["begin"], (sch, c["t"])
            assert list(rw["rows"][x]) == want["rows"], (sch, c["t"])


@pytest.mark.parametrize("mode", MODES)
def test_affine_scores_vs_oracle(gpu_engine, oracle, mode):
    rng = np.random.default_rng(300 + mode)
    schemes = [(1, -1, -2, -3), (2, -1, -1, -4), (1, 0, 0, -2), (5, -4, -1, -6), (7, -30, -20, -40), (1, -1, -2, -1)]
    for sch in schemes:
        trips = rand_trips(rng, 40, 0, 70) + rand_trips(rng, 8, 70, 170)
        out = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.affine(t, sch, mode)
            assert int(out["status"][x]) == 0
            assert int(out["score"][x]) == want["score"], (sch, mode, [len(s) for s in t])
            assert list(out["end"][x]) == want["end"], (sch, mode, [len(s) for s in t])


@pytest.mark.parametrize("mode", MODES)
def test_affine_rows_vs_oracle(gpu_engine, oracle, mode):
    rng = np.random.default_rng(400 + mode)
    for sch in [(1, -1, -2, -3), (2, -1, -1, -5), (3, -2, -1, -1)]:
        trips = rand_trips(rng, 30, 0, 50) + rand_trips(rng, 4, 75, 130)
        trips += [("", "", ""), ("A", "", ""), ("", "ACGT", "TTTT"), ("T" * 90, "", "A" * 85)]
        out = run(trips, sch, mode, rows=True)
        for x, t in enumerate(trips):
            want = oracle.affine(t, sch, mode, with_rows=True)
            assert int(out["status"][x]) == 0, (sch, mode, x)
            got = {"score": int(out["score"][x]), "end": list(out["end"][x]), "begin": list(out["begin"][x]),
                   "rows": list(out["rows"][x])}
            assert got == want, (sch, mode, [len(s) for s in t])


def test_affine_long_triplets_vs_oracle(gpu_engine, oracle):
    """Multi-block items (b, c beyond one 80-cell block, up to 4 x 4 blocks)."""
    rng = np.random.default_rng(7)
    trips = []
    for lens in [(170, 20, 30), (5, 200, 180), (30, 165, 330), (190, 161, 159), (0, 170, 170), (240, 250, 260)]:
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in lens))
    for mode in MODES:
        sch = (1, -1, -2, -3)
        out = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.affine(t, sch, mode)
            assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], (mode, x)


def test_affine_c2_sample_vs_oracle(gpu_engine, oracle):
    """Config C2 (150 bp, ~5% divergence): a prefix of the bench workload."""
    seqs, offs = oracle.generate("fixed:150:150:150:24", 0.025, 0.005, 2)
    sch = (1, -1, -2, -3)
    out = ta.align_arrays(seqs, offs, ta.ScoringScheme(*sch), ta.AlignmentMode.Global)
    rw = ta.align_arrays(seqs, offs, ta.ScoringScheme(*sch), ta.AlignmentMode.Global, with_rows=True,
                         cell_budget=1 << 40)
    for x in range(24):
        t = tuple(bytes(seqs[offs[3 * x + d]:offs[3 * x + d + 1]]).decode() for d in range(3))
        want = oracle.affine(t, sch, 0, with_rows=True)
        assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], x
        assert list(rw["rows"][x]) == want["rows"], x


def test_affine_invalid_open_rejected(gpu_engine):
    with pytest.raises(ta.InvalidArgument):
        ta.ScoringScheme(1, -1, -2, 3).validate()
    seqs, offs = trips_to_arrays([("ACGT", "ACGT", "ACGT")])
    with pytest.raises(ta.InvalidArgument):
        ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2, 5), ta.AlignmentMode.Global)


def test_cli_gap_open_matches_oracle(gpu_engine, oracle, tmp_path):
    """`trioalign align --gap-open` (the one added CLI flag) writes the
    affine scores of SPEC-AFFINE.md in the reference CSV format."""
    import os
    import subprocess
    rng = np.random.default_rng(21)
    trips = rand_trips(rng, 6, 5, 40)
    fa = tmp_path / "in.fa"
    with open(fa, "w") as f:
        for x, t in enumerate(trips):
            for d, s in enumerate(t):
                f.write(f">t{x}_{d}\n{s}\n")
    exe = os.path.join(os.path.dirname(ta.__file__), "trioalign")
    for mode, name in ((0, "global"), (1, "semiglobal"), (2, "local")):
        out = tmp_path / f"o{mode}.csv"
        p = subprocess.run([exe, "align", "--in", str(fa), "--out", str(out), "--mode", name, "--gap-open", "-3"],
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        lines = out.read_text().strip().splitlines()
        assert lines[0] == "id,mode,score,i,j,k,error"
        for x, line in enumerate(lines[1:]):
            f = line.split(",")
            want = oracle.affine(trips[x], (1, -1, -2, -3), mode)
            assert f[1] == name and int(f[2]) == want["score"] and [int(v) for v in f[3:6]] == want["end"], line


@pytest.mark.parametrize("mode", MODES)
def test_affine_wave_pairs_of_different_triplets(gpu_engine, oracle, mode):
    """Affine wave mode (few long triplets spread over all CTAs), pairing
    blocks of different triplets with equal a but different b, c."""
    rng = np.random.default_rng(77 + mode)
    trips = []
    for b, c in [(165, 300), (310, 170), (200, 200), (330, 161), (250, 180)]:
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in (180, b, c)))
    sch = (1, -1, -2, -3)
    out = run(trips, sch, mode)
    for x, t in enumerate(trips):
        want = oracle.affine(t, sch, mode)
        assert int(out["status"][x]) == 0
        assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], (mode, x)


@pytest.mark.parametrize("mode", MODES)
def test_affine_many_long_triplets_mixed_block_widths(gpu_engine, oracle, mode):
    """Enough long triplets to skip wave mode, b, c in 70..260: single-block
    items, 80-wide block items and 64-wide block items (4 x 4 tiles, chosen
    where they pad less, e.g. extents 81..128 and 193..256) vs the oracle."""
    rng = np.random.default_rng(600 + mode)
    trips = []
    for _ in range(320):
        a = int(rng.integers(0, 16))
        b, c = (int(x) for x in rng.integers(70, 261, size=2))
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in (a, b, c)))
    for sch in [(1, -1, -2, -3), (50, -50, -30, -40)]:  # the second one needs int32 lanes
        out = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.affine(t, sch, mode)
            assert int(out["status"][x]) == 0
            assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], (sch, mode, x)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_open_zero_equals_linear_on_mixed_block_grids(gpu_engine, mode):
    """Mixed lengths (C4-like, 64-512 bp): paired lanes whose first blocks
    look alike but whose block grids differ must not share packed faces.  With
    gap_open = 0 the forced affine kernels equal the linear kernels exactly."""
    ta = gpu_engine
    seqs, offs = ta.generate("uniform:64:512:3000", 0.08, 0.01, 4)
    lin = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode),
                          cfg=ta.EngineConfig(cell_budget=1 << 40))
    aff = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode),
                          cfg=ta.EngineConfig(cell_budget=1 << 40, gap_model=1))
    assert (lin["status"] == 0).all() and (aff["status"] == 0).all()
    bad = np.flatnonzero((lin["score"] != aff["score"]) | (lin["end"] != aff["end"]).any(axis=1))
    assert len(bad) == 0, bad[:10].tolist()


@pytest.mark.parametrize("mode", MODES)
def test_wave_traceback_vs_oracle(gpu_engine, oracle, mode):
    """Few long triplets take wave mode on the rows path too (their blocks
    spread over all CTAs, linear and affine kernels): score, end, begin and
    rows equal the oracles'."""
    rng = np.random.default_rng(31)
    base = "".join("ACGT"[x] for x in rng.integers(0, 4, size=260))
    def mutate(s):
        return "".join(("ACGT"[rng.integers(0, 4)] if rng.random() < 0.08 else c) for c in s if rng.random() > 0.02)
    trips = [(mutate(base[:230]), mutate(base[:250]), mutate(base[:220])), (mutate(base), mutate(base[:200]), mutate(base))]
    for sch in ((1, -1, -2, 0), (1, -1, -2, -3)):
        out = run(trips, sch, mode, rows=True)
        for x, t in enumerate(trips):
            want = (oracle.align(t, sch[:3], mode, with_rows=True) if sch[3] == 0
                    else oracle.affine(t, sch, mode, with_rows=True))
            got = {"score": int(out["score"][x]), "end": [int(v) for v in out["end"][x]],
                   "begin": [int(v) for v in out["begin"][x]], "rows": list(out["rows"][x])}
            assert got == want, (sch, mode, x)
