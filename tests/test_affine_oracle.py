"""Pinning the affine-gap oracle (SPEC-AFFINE.md; the reference has no affine
gaps, so parity for affine is against this definition):

1. gap_open = 0 reproduces the reference's own linear results (golden
   vectors made by oracle/_ref) - scores and end coordinates;
2. an independent exhaustive enumerator of every 3-way alignment of small
   triplets, scored column by column, agrees with the oracle's DP;
3. every traceback rescored with the column rule gives the reported score
   and strips back to the inputs.
CPU only."""
import itertools
import random

import pytest

from conftest import load_golden

GAP = "-"
MASKS = {1: 7, 2: 3, 3: 5, 4: 6, 5: 1, 6: 2, 7: 4}  # column type -> residue mask (bit 0 = s0)
PAIRS = ((0, 1), (0, 2), (1, 2))


def pair_state(mask, p, q):
    rp, rq = (mask >> p) & 1, (mask >> q) & 1
    return "M" if rp and rq else "P" if rp else "Q" if rq else "N"


def sigma(x, y, sch):
    if x == GAP and y == GAP:
        return 0
    if x == GAP or y == GAP:
        return sch[2]
    return sch[0] if x == y else sch[1]


def column_score(cols, prev_mask, sch):
    """cols: the three characters; prev_mask: residue mask of the previous column."""
    mask = sum(1 << d for d in range(3) if cols[d] != GAP)
    s = 0
    for p, q in PAIRS:
        s += sigma(cols[p], cols[q], sch)
        st = pair_state(mask, p, q)
        if st in "PQ" and pair_state(prev_mask, p, q) != st:
            s += sch[3]
    return s, mask


def brute_force(t, sch, mode):
    """Max over all alignments (every start / end the mode allows) and the
    lexicographically smallest end attaining it - by enumeration, no DP."""
    a, b, c = (len(x) for x in t)
    cells = [(i, j, k) for i in range(a + 1) for j in range(b + 1) for k in range(c + 1)]

    def is_start(i, j, k):
        z = (i == 0) + (j == 0) + (k == 0)
        return z == 3 if mode == 0 else z >= 2 if mode == 1 else True

    def is_end(i, j, k):
        return (i, j, k) == (a, b, c) if mode == 0 else (i == a or j == b or k == c) if mode == 1 else True

    best = {}

    def dfs(i, j, k, prev_mask, score):
        if is_end(i, j, k) and score > best.get((i, j, k), -10 ** 9):
            best[(i, j, k)] = score
        for t_ in range(1, 8):
            m = MASKS[t_]
            ni, nj, nk = i + (m & 1), j + ((m >> 1) & 1), k + ((m >> 2) & 1)
            if ni > a or nj > b or nk > c:
                continue
            cols = (t[0][i] if m & 1 else GAP, t[1][j] if m & 2 else GAP, t[2][k] if m & 4 else GAP)
            cs, mask = column_score(cols, prev_mask, sch)
            dfs(ni, nj, nk, mask, score + cs)

    for st in cells:
        if is_start(*st):
            dfs(*st, 7, 0)
    top = max(best.values())
    end = min(e for e, v in best.items() if v == top)
    return top, list(end)


def rand_seq(rng, n):
    return "".join(rng.choice("ACGT") for _ in range(n))


@pytest.mark.parametrize("mode", (0, 1, 2))
def test_open_zero_is_the_reference_linear_model(oracle, mode):
    cases = [c for c in load_golden("small_rows.json.gz") if c["mode"] == mode]
    assert cases
    for c in cases[:150]:
        sch = tuple(c["scheme"]) + (0,)
        got = oracle.affine(c["t"], sch, mode)
        assert got["score"] == c["oracle"]["score"], c
        assert got["end"] == c["oracle"]["end"], c


def test_open_zero_kats(oracle):
    for case in load_golden("kat.json"):
        got = oracle.affine(case["t"], tuple(case["scheme"]) + (0,), case["mode"])
        assert got["score"] == case["oracle"]["score"] and got["end"] == case["oracle"]["end"], case


@pytest.mark.parametrize("mode", (0, 1, 2))
def test_dp_equals_exhaustive_enumeration(oracle, mode):
    rng = random.Random(17 + mode)
    schemes = [(1, -1, -2, -3), (2, -1, -1, -4), (1, 0, 0, -1), (3, -2, -1, 0), (1, -1, -2, -10), (5, -4, -2, -2)]
    maxlen = 3 if mode < 2 else 2
    for sch in schemes:
        for _ in range(6):
            t = tuple(rand_seq(rng, rng.randint(0, maxlen)) for _ in range(3))
            want_score, want_end = brute_force(t, sch, mode)
            got = oracle.affine(t, sch, mode)
            assert got["score"] == want_score, (t, sch, mode)
            assert got["end"] == want_end, (t, sch, mode)
    # all length combinations of two identical / mismatching bases
    for lens in itertools.product(range(3), repeat=3):
        t = tuple(("AC" * 2)[:L] if d != 1 else ("AG" * 2)[:L] for d, L in enumerate(lens))
        want = brute_force(t, (1, -1, -2, -3), mode)
        got = oracle.affine(t, (1, -1, -2, -3), mode)
        assert (got["score"], got["end"]) == want, (t, mode)


@pytest.mark.parametrize("mode", (0, 1, 2))
def test_traceback_rescores_to_the_score(oracle, mode):
    rng = random.Random(5 + mode)
    for sch in [(1, -1, -2, -3), (2, -1, -1, -5), (1, 0, 0, -2), (3, -2, -1, 0)]:
        for _ in range(40):
            t = tuple(rand_seq(rng, rng.randint(0, 14)) for _ in range(3))
            got = oracle.affine(t, sch, mode, with_rows=True)
            rows = got["rows"]
            assert len({len(r) for r in rows}) == 1
            bi, bj, bk = got["begin"]
            ei, ej, ek = got["end"]
            # semi-global: free prefix / suffix columns lie outside the scored span
            lo = bi + bj + bk if mode == 1 else 0
            hi = len(rows[0]) - ((len(t[0]) - ei) + (len(t[1]) - ej) + (len(t[2]) - ek) if mode == 1 else 0)
            assert oracle.affine_rescore(rows, lo, hi, sch) == got["score"], (t, sch, mode, rows)
            if mode == 0:
                for d in range(3):
                    assert rows[d].replace(GAP, "") == t[d]
            else:
                b_, e_ = got["begin"], got["end"]
                for d in range(3):
                    want = t[d] if mode == 1 else t[d][b_[d]:e_[d]]
                    assert rows[d].replace(GAP, "") == want, (t, rows, mode)


def test_affine_open_penalises_fragmented_gaps(oracle):
    # one 3-residue gap run in s1 beats three separate gaps once opening costs
    t = ("AAACCCGGG", "AAAGGG", "AAACCCGGG")
    lin = oracle.affine(t, (2, -1, -1, 0), 0, with_rows=True)
    aff = oracle.affine(t, (2, -1, -1, -4), 0, with_rows=True)
    assert aff["score"] <= lin["score"]
    assert "---" in aff["rows"][1]
