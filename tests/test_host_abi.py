"""C-ABI library loads and exports every symbol include/trioalign_capi.h
declares; host-side helpers keep the reference semantics.  CPU only (no
compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2605_28400_b200 as ta

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "trioalign_capi.h")).read()
    return sorted(set(re.findall(r"\b(ta_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ta.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(ta.EXPORTED_SYMBOLS) <= set(syms)


def test_version_and_device_count_do_not_crash():
    assert b"sm_100a" in ta.lib().ta_version()
    assert ta.device_count() >= 0


def test_compute_without_gpu_fails_loudly():
    if ta.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(ta.CudaError):
        ta.align(ta.Triplet("t", "ACGT", "ACG", "AC"), ta.ScoringScheme(), ta.AlignmentMode.Global,
                 ta.EngineConfig())


# --- plan_partition: test_dispatch.cpp:35-115 / SPEC.md:269-274 ------------

def test_partition_blocked_interleaved_dynamic():
    assert ta.plan_partition([1] * 5, ta.Strategy.Blocked, 2).assignment == [0, 0, 0, 1, 1]
    assert ta.plan_partition([1] * 5, ta.Strategy.Interleaved, 2).assignment == [0, 1, 0, 1, 0]
    assert ta.plan_partition([100, 1, 1, 1], ta.Strategy.Dynamic, 2).assignment == [0, 1, 1, 1]
    assert ta.plan_partition([5, 5, 5, 5], ta.Strategy.Dynamic, 3).assignment == [0, 1, 2, 0]


def test_partition_errors():
    with pytest.raises(ta.ConfigError):
        ta.plan_partition([1, 2], ta.Strategy.Blocked, 0)
    with pytest.raises(ta.ConfigError):
        ta.plan_partition([], ta.Strategy.Blocked, 2)


def test_partition_greedy_bound():
    import random
    rnd = random.Random(3)
    for w in (1, 2, 3, 5, 8):
        cells = [rnd.randrange(1, 10000) for _ in range(200)]
        plan = ta.plan_partition(cells, ta.Strategy.Dynamic, w)
        loads = [0] * w
        for c, a in zip(cells, plan.assignment):
            loads[a] += c
        assert max(loads) <= sum(cells) / w + max(cells)


def test_strategy_names_round_trip():
    for s in ta.Strategy:
        assert ta.strategy_from_name(ta.strategy_name(s)) == s
    with pytest.raises(ta.ParseError):
        ta.strategy_from_name("stealing")


# --- tiled.cpp helpers / validation -----------------------------------------

def test_packed_score_bound_formula():  # test_tiled.cpp:277-282
    t = ta.Triplet("t", "ACGT", "ACG", "AC")
    assert ta.packed_score_bound(t, ta.ScoringScheme(1, -1, -2)) == 36
    assert ta.packed_score_bound(t, ta.ScoringScheme(5, -1, -2)) == 135
    assert ta.packed_score_bound(t, ta.ScoringScheme(1, -1, -300)) == 5400
    sch = ta._Scheme(1, -1, -300)
    assert ta.lib().ta_packed_score_bound(4, 3, 2, ctypes.byref(sch)) == 5400
    big = ta.Triplet("big", "A" * 32, "A" * 32, "A" * 32)
    assert not ta.packed_bound_ok(big, ta.ScoringScheme(5, -1, -300))
    assert ta.packed_bound_ok(big, ta.ScoringScheme(1, -1, -2))


def test_derive_team_width():
    for n, b, c in [(8, 0, 0), (8, 7, 3), (8, 8, 9), (16, 150, 149), (3, 10, 2)]:
        assert ta.lib().ta_derive_team_width(n, b, c) == ta.derive_team_width(n, b, c)


def test_scheme_validation():
    for bad in [(0, -1, -2), (1, 1, -2), (1, -1, 2), (1025, -1, -2)]:
        with pytest.raises(ta.InvalidArgument):
            ta.make_scheme(*bad)
        assert ta.lib().ta_validate_scheme(ctypes.byref(ta._Scheme(*bad))) == 7
    assert ta.lib().ta_validate_scheme(ctypes.byref(ta._Scheme(1, -1, -2))) == 0


def test_affine_scheme_validation():  # SPEC-AFFINE.md: gap_open <= 0, |gap_open| <= 1024
    for bad in [(1, -1, -2, 1), (1, -1, -2, -1025)]:
        with pytest.raises(ta.InvalidArgument):
            ta.ScoringScheme(*bad).validate()
        assert ta.lib().ta_validate_scheme(ctypes.byref(ta._Scheme(*bad))) == 7
    ta.ScoringScheme(1, -1, -2, -3).validate()
    assert ta.lib().ta_validate_scheme(ctypes.byref(ta._Scheme(1, -1, -2, -3))) == 0
    # the C-ABI structs match the header (4 x int32 scheme; options end with gap_model)
    assert ctypes.sizeof(ta._Scheme) == 16
    assert [f for f, _ in ta._Options._fields_][-1] == "gap_model"


def test_engine_config_validation():
    with pytest.raises(ta.ConfigError):
        ta.EngineConfig(tile_size=0).validate()
    opt = ta._options(0, False, ta.EngineConfig(tile_size=5000))
    assert ta.lib().ta_validate_options(ctypes.byref(opt)) == 3
    opt = ta._options(0, False, ta.EngineConfig())
    assert ta.lib().ta_validate_options(ctypes.byref(opt)) == 0


def test_mode_names():
    for m in ta.AlignmentMode:
        assert ta.mode_from_name(ta.mode_name(m)) == m
    with pytest.raises(ta.ParseError):
        ta.mode_from_name("glocal")


def test_sigma_sop_kats():  # test_core.cpp / SPEC.md examples
    s = ta.ScoringScheme(1, -1, -2)
    assert ta.sigma("A", "A", s) == 1 and ta.sigma("A", "C", s) == -1
    assert ta.sigma("A", "-", s) == -2 and ta.sigma("-", "-", s) == 0
    assert ta.sop("A", "A", "A", s) == 3 and ta.sop("A", "-", "-", s) == -4
    assert ta.sop("A", "C", "-", s) == -5
