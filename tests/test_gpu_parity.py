"""GPU parity: the sm_100a kernels (through the C-ABI) against the oracle and
the reference's own golden vectors.  Bit-exact (integer DP).  Needs a B200."""
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


def run(trips, scheme, mode, rows=False):
    seqs, offs = trips_to_arrays(trips)
    return ta.align_arrays(seqs, offs, ta.ScoringScheme(*scheme), ta.AlignmentMode(mode),
                           with_rows=rows, cell_budget=(1 << 40) if rows else None)


def test_kat(gpu_engine):
    for case in load_golden("kat.json"):
        out = run([case["t"]], case["scheme"], case["mode"], rows=True)
        want = case["oracle"]
        assert int(out["status"][0]) == 0
        assert int(out["score"][0]) == want["score"], case
        assert list(out["end"][0]) == want["end"], case
        assert list(out["begin"][0]) == want["begin"], case
        assert list(out["rows"][0]) == want["rows"], case


@pytest.mark.parametrize("mode", MODES)
def test_small_corpus_scores_and_rows(gpu_engine, mode):
    cases = [c for c in load_golden("small_rows.json.gz") if c["mode"] == mode]
    by_scheme = {}
    for c in cases:
        by_scheme.setdefault(tuple(c["scheme"]), []).append(c)
    for sch, cs in by_scheme.items():
        trips = [c["t"] for c in cs]
        score_only = run(trips, sch, mode)
        with_rows = run(trips, sch, mode, rows=True)
        for x, c in enumerate(cs):
            want = c["oracle"]
            assert int(score_only["status"][x]) == 0
            assert int(score_only["score"][x]) == want["score"], (sch, c["t"])
            assert list(score_only["end"][x]) == want["end"], (sch, c["t"])
            assert int(with_rows["score"][x]) == want["score"]
            assert list(with_rows["end"][x]) == want["end"]
            assert list(with_rows["begin"][x]) == want["begin"], (sch, c["t"])
            assert list(with_rows["rows"][x]) == want["rows"], (sch, c["t"])


def test_c1_all_rows_global(gpu_engine):
    c1 = load_golden("c1_rows.json.gz")
    from oracle.pyoracle import Oracle
    seqs, offs = Oracle().generate(c1["spec"], c1["rates"][0], c1["rates"][1], c1["seed"])
    for mode, recs in c1["modes"].items():
        n = len(recs)
        out = ta.align_arrays(seqs, offs[:3 * n + 1], ta.ScoringScheme(*c1["scheme"]),
                              ta.AlignmentMode(int(mode)), with_rows=True, cell_budget=1 << 40)
        sc = ta.align_arrays(seqs, offs[:3 * n + 1], ta.ScoringScheme(*c1["scheme"]),
                             ta.AlignmentMode(int(mode)))
        for t in range(n):
            w = recs[t]
            assert int(out["score"][t]) == w["score"] and int(sc["score"][t]) == w["score"], t
            assert list(out["end"][t]) == w["end"] and list(sc["end"][t]) == w["end"], t
            assert list(out["begin"][t]) == w["begin"], t
            assert list(out["rows"][t]) == w["rows"], t


@pytest.mark.parametrize("mode", MODES)
def test_random_vs_oracle_many_lengths(gpu_engine, oracle, mode):
    rng = np.random.default_rng(1234 + mode)
    for sch in [(1, -1, -2), (2, -1, -2), (3, -2, -1), (1, 0, 0), (5, -4, -1), (7, -30, -20)]:
        trips = []
        for _ in range(60):
            lens = rng.integers(0, 60, size=3)
            if rng.random() < 0.2:
                lens = rng.integers(90, 159, size=3)
            trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in lens))
        out = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.align(t, sch, mode)
            assert int(out["status"][x]) == 0
            assert int(out["score"][x]) == want["score"], (sch, mode, t)
            assert list(out["end"][x]) == want["end"], (sch, mode, t)


def test_config_samples_vs_reference(gpu_engine, oracle):
    cfgs = load_golden("configs.json.gz")
    for name in ("C2", "C3"):
        ent = cfgs[name]
        seqs, offs = oracle.generate(ent["sample_spec"], ent["rates"][0], ent["rates"][1], ent["seed"])
        for mode, recs in ent["modes"].items():
            n = len(recs)
            out = ta.align_arrays(seqs, offs[:3 * n + 1], ta.ScoringScheme(*ent["scheme"]),
                                  ta.AlignmentMode(int(mode)))
            for t in range(n):
                assert int(out["score"][t]) == recs[t]["score"], (name, mode, t)
                assert list(out["end"][t]) == recs[t]["end"], (name, mode, t)
        if "rows_global" in ent:
            k = len(ent["rows_global"])
            out = ta.align_arrays(seqs, offs[:3 * k + 1], ta.ScoringScheme(*ent["scheme"]),
                                  ta.AlignmentMode.Global, with_rows=True, cell_budget=1 << 40)
            for t in range(k):
                assert list(out["rows"][t]) == ent["rows_global"][t]["rows"], (name, t)


def test_reference_api_errors(gpu_engine):
    t = ta.Triplet("t", "ACGTACGT", "ACGTACGT", "ACGTACGT")
    cfg = ta.EngineConfig(tile_size=4, cell_budget=10)
    with pytest.raises(ta.CapacityError):
        ta.align(t, ta.ScoringScheme(), ta.AlignmentMode.Global, cfg)
    with pytest.raises(ta.ConfigError):
        ta.align(t, ta.ScoringScheme(), ta.AlignmentMode.Global, ta.EngineConfig(tile_size=2, team_width=2))
    a = ta.Triplet("a", "ACGT", "AC", "G")
    b = ta.Triplet("b", "ACG", "AC", "G")
    with pytest.raises(ta.ShapeMismatchError):
        ta.align_packed(a, b, ta.ScoringScheme(), ta.AlignmentMode.Global, ta.EngineConfig(tile_size=4))
    big = ta.Triplet("big", "A" * 32, "A" * 32, "A" * 32)
    with pytest.raises(ta.LaneOverflowError):
        ta.align_packed(big, big, ta.ScoringScheme(5, -1, -300), ta.AlignmentMode.Global, ta.EngineConfig())
    with pytest.raises(ta.CapacityError):
        ta.oracle_align(ta.Triplet("big", "ACGTACGT", "ACGTACGT", "ACGTACGT"), ta.ScoringScheme(),
                        ta.AlignmentMode.Global, True, 100)
    r = ta.align(ta.Triplet("id", "ACG", "ACG", "ACG"), ta.ScoringScheme(2, -1, -2),
                 ta.AlignmentMode.Global, ta.EngineConfig(tile_size=2))
    assert r.score == 18 and r.end == (3, 3, 3)


def test_run_batch_failures_recorded(gpu_engine):
    data = [ta.Triplet(f"t{i}", "ACGT", "ACGA", "AGGT") for i in range(3)]
    data.insert(1, ta.Triplet("too-big", "A" * 40, "A" * 40, "A" * 40))
    cells = [t.cell_count() for t in data]
    cfg = ta.EngineConfig(tile_size=4, cell_budget=10000)
    rep = ta.run_batch(data, ta.ScoringScheme(), ta.AlignmentMode.Global, cfg,
                       ta.plan_partition(cells, ta.Strategy.Interleaved, 2))
    assert [o.ok for o in rep.per_triplet] == [True, False, True, True]
    assert "budget" in rep.per_triplet[1].error
    assert rep.scored_cells == sum(o.cells for o in rep.per_triplet if o.ok)


def test_empty_and_degenerate(gpu_engine):
    trips = [("", "", ""), ("A", "", ""), ("", "C", ""), ("", "", "G"), ("ACGT", "", ""),
             ("", "ACGT", "TTTT"), ("A", "A", ""), ("T" * 150, "", "A" * 150)]
    from oracle.pyoracle import Oracle
    o = Oracle()
    for mode in MODES:
        out = run(trips, (1, -1, -2), mode, rows=True)
        for x, t in enumerate(trips):
            want = o.align(t, (1, -1, -2), mode, with_rows=True)
            assert int(out["score"][x]) == want["score"], (mode, t)
            assert list(out["end"][x]) == want["end"], (mode, t)
            assert list(out["rows"][x]) == want["rows"], (mode, t)


@pytest.mark.parametrize("mode", MODES)
def test_c4_mixed_long_vs_reference(gpu_engine, oracle, mode):
    """Mixed 64-512 bp (config C4): multi-block items through global faces."""
    ent = load_golden("configs.json.gz")["C4"]
    seqs, offs = oracle.generate(ent["sample_spec"], ent["rates"][0], ent["rates"][1], ent["seed"])
    recs = ent["modes"][str(mode)]
    n = len(recs)
    out = ta.align_arrays(seqs, offs[:3 * n + 1], ta.ScoringScheme(*ent["scheme"]), ta.AlignmentMode(mode))
    for t in range(n):
        assert int(out["status"][t]) == 0, t
        assert int(out["score"][t]) == recs[t]["score"], (mode, t, ent["lengths"][t])
        assert list(out["end"][t]) == recs[t]["end"], (mode, t, ent["lengths"][t])


@pytest.mark.parametrize("mode", MODES)
def test_long_random_rows_vs_oracle(gpu_engine, oracle, mode):
    """Ragged long triplets (b or c beyond one 160-cell block, a < G), rows too."""
    rng = np.random.default_rng(99 + mode)
    trips = []
    for lens in [(170, 20, 30), (5, 200, 180), (30, 165, 330), (190, 161, 159), (2, 321, 9), (0, 170, 170),
                 (161, 0, 161), (240, 250, 260)]:
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in lens))
    for sch in [(1, -1, -2), (3, -2, -1)]:
        out = run(trips, sch, mode, rows=True)
        sc = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.align(t, sch, mode, with_rows=True)
            assert int(out["status"][x]) == 0 and int(sc["status"][x]) == 0
            assert int(sc["score"][x]) == want["score"] and list(sc["end"][x]) == want["end"], (sch, mode, x)
            assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], (sch, mode, x)
            assert list(out["begin"][x]) == want["begin"], (sch, mode, x)
            assert list(out["rows"][x]) == want["rows"], (sch, mode, x)


def test_c5_single_long_triplets_vs_reference(gpu_engine, oracle):
    """Config C5: single 1000 / 1500 / 2000 bp triplets (one stream, 7x7 to 13x13
    blocks), global score and end vs the reference tiled engine."""
    cfgs = load_golden("configs.json.gz")
    for name in ("C5a", "C5b", "C5c"):
        ent = cfgs[name]
        seqs, offs = oracle.generate(ent["sample_spec"], ent["rates"][0], ent["rates"][1], ent["seed"])
        out = ta.align_arrays(seqs, offs, ta.ScoringScheme(*ent["scheme"]), ta.AlignmentMode.Global,
                              cfg=ta.EngineConfig(cell_budget=1 << 40))
        want = ent["modes"]["0"][0]
        assert int(out["status"][0]) == 0, name
        assert int(out["score"][0]) == want["score"], name
        assert list(out["end"][0]) == want["end"], name


@pytest.mark.parametrize("mode", MODES)
def test_wave_pairs_of_different_triplets(gpu_engine, oracle, mode):
    """Wave mode (few long triplets spread over all CTAs) pairing blocks of
    DIFFERENT triplets with equal a but different b, c in the two lanes: a
    tile can be padding for one lane and real for the other."""
    rng = np.random.default_rng(55 + mode)
    trips = []
    for b, c in [(165, 300), (310, 170), (200, 200), (330, 161), (161, 330), (250, 180)]:
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in (180, b, c)))
    out = run(trips, (1, -1, -2), mode)
    for x, t in enumerate(trips):
        want = oracle.align(t, (1, -1, -2), mode)
        assert int(out["status"][x]) == 0
        assert int(out["score"][x]) == want["score"] and list(out["end"][x]) == want["end"], (mode, x)


@pytest.mark.parametrize("mode", MODES)
def test_many_long_triplets_mixed_block_widths(gpu_engine, oracle, mode):
    """Enough long triplets to skip wave mode (> one per two lane streams), with
    b, c in 150..300: the largest-grid bucket splits into single-block items,
    160-wide block items and 128-wide block items (8 x 8 tiles, chosen where
    they pad less, e.g. extents 161..256); every score and end vs the oracle."""
    rng = np.random.default_rng(500 + mode)
    trips = []
    for _ in range(320):
        a = int(rng.integers(0, 24))
        b, c = (int(x) for x in rng.integers(150, 301, size=2))
        trips.append(tuple("".join("ACGT"[x] for x in rng.integers(0, 4, size=L)) for L in (a, b, c)))
    for sch in [(1, -1, -2), (2, -3, -1), (100, -100, -50)]:  # the last one needs int32 lanes
        sc = run(trips, sch, mode)
        for x, t in enumerate(trips):
            want = oracle.align(t, sch, mode)
            assert int(sc["status"][x]) == 0
            assert int(sc["score"][x]) == want["score"] and list(sc["end"][x]) == want["end"], (sch, mode, x)


def test_device_batch_rerun_cache(gpu_engine):
    """A resident batch re-run with the same scheme/options reuses its host
    plan (front cache); any change of scheme, mode, options or an affine /
    rows run in between must re-plan.  Every run equals a fresh one-shot run."""
    seqs, offs = ta.generate("uniform:40:170:600", 0.05, 0.01, 21)
    b = ta.DeviceBatch(seqs, offs)
    seq = [((1, -1, -2, 0), 0), ((1, -1, -2, 0), 0), ((1, -1, -2, 0), 1), ((2, -1, -1, 0), 1),
           ((1, -1, -2, -3), 0), ((1, -1, -2, 0), 1), ((1, -1, -2, 0), 2), ((1, -1, -2, 0), 2),
           ((1, -1, -2, 0), 0)]
    for sch, mode in seq:
        b.run(ta.ScoringScheme(*sch), ta.AlignmentMode(mode), ta.EngineConfig(cell_budget=1 << 40))
        got = b.fetch()
        want = ta.align_arrays(seqs, offs, ta.ScoringScheme(*sch), ta.AlignmentMode(mode), cell_budget=1 << 40)
        assert (got["status"] == want["status"]).all(), (sch, mode)
        assert (got["score"] == want["score"]).all(), (sch, mode)
        assert (got["end"] == want["end"]).all(), (sch, mode)
    # an option change that fails every triplet, then the valid options again
    b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1))
    assert (b.fetch()["status"] != 0).all()
    b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(0), ta.EngineConfig(cell_budget=1 << 40))
    assert (b.fetch()["status"] == 0).all()


def test_one_shot_statuses_across_chunks(gpu_engine):
    """The pipelined one-shot path (ta_align_batch, ~10 chunks here) checks
    and packs each chunk behind the previous chunk's kernels: per-triplet
    statuses (non-ACGT residues, cell budget) and results must equal the
    resident-batch path's on the same inputs; malformed offsets fail the call."""
    seqs, offs = ta.generate("uniform:20:150:200000", 0.05, 0.01, 23)
    seqs = seqs.copy()
    n = (len(offs) - 1) // 3
    for t in (5, 77777, 150001, n - 1):  # a residue 'N' in four chunks
        seqs[offs[3 * t + 1]] = ord("N")
    lens = np.diff(offs).reshape(-1, 3).astype(np.int64)
    budget = int(np.percentile(np.prod(lens, axis=1), 90))  # ~10% capacity errors
    for mode in (0, 1):
        cfg = ta.EngineConfig(cell_budget=budget)
        got = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), cfg=cfg)
        b = ta.DeviceBatch(seqs, offs)
        b.run(ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode), cfg)
        want = b.fetch()
        assert (got["status"] == want["status"]).all(), mode
        assert (got["score"] == want["score"]).all() and (got["end"] == want["end"]).all(), mode
        assert int((got["status"] != 0).sum()) > n // 20
        assert all(int(got["status"][t]) != 0 for t in (5, 77777, 150001, n - 1))
    bad = offs.copy()
    bad[3 * 1000 + 1] = bad[3 * 1000] - 1  # a negative length
    with pytest.raises(Exception):
        ta.align_arrays(seqs, bad, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode.Global)
