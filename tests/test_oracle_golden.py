"""The oracle (C restatement, oracle/trio_oracle.c) pinned against fixtures
produced by the reference itself (tests/golden/make_golden.py over
oracle/_ref).  CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden


def test_kat(oracle):
    for case in load_golden("kat.json"):
        got = oracle.align(case["t"], case["scheme"], case["mode"], with_rows=True)
        assert got == case["oracle"], case


def test_small_corpus_rows(oracle):
    cases = load_golden("small_rows.json.gz")
    assert len(cases) == 720
    for case in cases:
        got = oracle.align(case["t"], case["scheme"], case["mode"], with_rows=True)
        assert got == case["oracle"], case
        # the reference tiled engine agrees with its oracle (test_tiled.cpp:112-132)
        assert case["tiled"]["score"] == got["score"] and case["tiled"]["end"] == got["end"]


def test_c1_rows_prefix(oracle):
    c1 = load_golden("c1_rows.json.gz")
    seqs, offs = oracle.generate(c1["spec"], c1["rates"][0], c1["rates"][1], c1["seed"])
    for mode, recs in c1["modes"].items():
        for t in range(0, len(recs), 25 if mode == "0" else 10):
            trip = [bytes(seqs[offs[3 * t + d]:offs[3 * t + d + 1]]).decode() for d in range(3)]
            assert oracle.align(trip, c1["scheme"], int(mode), with_rows=True) == recs[t]


@pytest.mark.parametrize("name", ["C1", "C4", "uniform:0:12:300", "blocked:5,9,20:30",
                                  "cycle:3,17,8:31", "fixed:4:7:2:5"])
def test_generator_restatement_matches_reference(oracle, name):
    h = load_golden("gen_hashes.json")[name]
    seqs, offs = oracle.generate(h["spec"], h["rates"][0], h["rates"][1], h["seed"])
    assert hashlib.sha256(seqs.tobytes()).hexdigest() == h["sha256_seqs"]
    assert hashlib.sha256(offs.astype("<i8").tobytes()).hexdigest() == h["sha256_offsets"]


def test_config_samples(oracle):
    cfgs = load_golden("configs.json.gz")
    for name in ("C2", "C3"):
        ent = cfgs[name]
        seqs, offs = oracle.generate(ent["sample_spec"], ent["rates"][0], ent["rates"][1], ent["seed"])
        for t in range(min(4, len(ent["lengths"]))):
            trip = [bytes(seqs[offs[3 * t + d]:offs[3 * t + d + 1]]).decode() for d in range(3)]
            want = ent["modes"]["0"][t]
            got = oracle.align(trip, ent["scheme"], 0)
            assert got == want, (name, t)
