"""Full-size parity properties (BASELINE.json configs at their real sizes,
where the CPU oracle cannot follow): size-independent invariants of the
reference semantics (SPEC.md oracle module) checked on every triplet.

* mode ordering: local >= semi-global >= global for match >= 0 >= mismatch, gap
  (pointwise tensor dominance + superset extraction regions);
* permutation invariance: permuting the three sequences leaves the score
  unchanged (and permutes the end coordinates in global mode);
* two independent kernel families agree: the affine kernels forced with
  gap_open = 0 reproduce the linear kernels' scores and ends bit for bit;
* s16x2 and int32 lanes agree (a scheme scaled so the host must pick int32
  lanes gives exactly the scaled scores);
* the CPU reference itself on a strided sample.
Needs a B200."""
import numpy as np
import pytest

import paper_2605_28400_b200 as ta

pytestmark = pytest.mark.gpu

C2 = ("fixed:150:150:150:1000000", (0.025, 0.005), 2)


@pytest.fixture(scope="module")
def c2():
    seqs, offs = ta.generate(C2[0], *C2[1], C2[2])
    return seqs, offs


def scores(seqs, offs, mode, sch=(1, -1, -2), force_affine=False):
    out = ta.align_arrays(seqs, offs, ta.ScoringScheme(*sch), ta.AlignmentMode(mode),
                          cfg=ta.EngineConfig(cell_budget=1 << 40, gap_model=1 if force_affine else 0))
    assert int((out["status"] != 0).sum()) == 0
    return out


def test_c2_full_mode_ordering(gpu_engine, c2):
    g = scores(*c2, 0)["score"]
    s = scores(*c2, 1)["score"]
    loc = scores(*c2, 2)["score"]
    assert len(g) == 1000000
    assert (loc >= s).all() and (s >= g).all()


def test_c2_full_permutation_invariance(gpu_engine, c2):
    seqs, offs = c2
    n = (len(offs) - 1) // 3
    base = scores(seqs, offs, 0)
    # rotate (s0, s1, s2) -> (s1, s2, s0): new offsets over the same buffer order
    lens = np.diff(offs).reshape(n, 3)
    starts = offs[:-1].reshape(n, 3)
    perm = [1, 2, 0]
    # build the rotated buffer vectorised: gather byte ranges in the new order
    order_starts = starts[:, perm].reshape(-1)
    order_lens = lens[:, perm].reshape(-1)
    idx = np.repeat(order_starts - np.concatenate([[0], np.cumsum(order_lens)[:-1]]), order_lens) + \
        np.arange(int(order_lens.sum()))
    rot = np.concatenate([seqs[:int(offs[-1])][idx], np.zeros(1, np.uint8)])
    roff = np.concatenate([[0], np.cumsum(order_lens)]).astype(np.int64)
    got = scores(rot, roff, 0)
    assert np.array_equal(got["score"], base["score"])
    assert np.array_equal(got["end"], base["end"][:, perm])


def test_affine_kernels_at_open_zero_equal_linear_kernels(gpu_engine, c2):
    seqs, offs = c2
    m = 200000
    o = offs[:3 * m + 1]
    for mode in (0, 1, 2):
        lin = scores(seqs, o, mode)
        aff = scores(seqs, o, mode, sch=(1, -1, -2, 0), force_affine=True)
        assert np.array_equal(lin["score"], aff["score"]), mode
        assert np.array_equal(lin["end"], aff["end"]), mode


def test_int32_and_s16_lanes_agree_at_scale(gpu_engine, c2):
    """(k, -k, -2k) scores are exactly k x (1, -1, -2); at k = 40 the host
    cannot prove the s16 bound and switches to int32 lanes."""
    seqs, offs = c2
    m = 100000
    o = offs[:3 * m + 1]
    for mode in (0, 2):
        a = scores(seqs, o, mode)
        b = scores(seqs, o, mode, sch=(40, -40, -80))
        assert np.array_equal(a["score"] * 40, b["score"]), mode
        assert np.array_equal(a["end"], b["end"]), mode


def test_c2_strided_sample_vs_reference(gpu_engine, oracle):
    """Every 2000th triplet of the full C2 batch against the CPU restatement
    (pinned to the reference): 500 triplets spread over the whole batch."""
    seqs, offs = ta.generate(C2[0], *C2[1], C2[2])
    out = scores(seqs, offs, 0)
    for t in range(0, 1000000, 2000):
        trip = tuple(bytes(seqs[offs[3 * t + d]:offs[3 * t + d + 1]]).decode() for d in range(3))
        want = oracle.align(trip, (1, -1, -2), 0)
        assert int(out["score"][t]) == want["score"] and list(out["end"][t]) == want["end"], t
