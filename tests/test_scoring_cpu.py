"""CPU: the §8(f) "next" rows -- the direct-form baseline and evaluate
restated in the oracle, and the constant-shift fixtures -- pinned to golden
vectors from the real reference (tools/make_golden.py scoring_cases)."""

import os

import numpy as np
import pytest

from oracle import mshbm_oracle as O

from mshbm_testutil import GOLDEN


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "scoring.npz"))


def test_shifted_pair_and_mask_match_reference(g):
    from paper_1901_09593_b200.synthetic import interior_mask, shifted_pair
    left, right = shifted_pair(24, 40, 4, np.random.default_rng(31), cutoff=0.15)
    np.testing.assert_array_equal(left, g["sp_left"])
    np.testing.assert_array_equal(right, g["sp_right"])
    np.testing.assert_array_equal(interior_mask(left.shape, 4, 5), g["sp_mask"])
    np.testing.assert_array_equal(interior_mask((30, 41), 3, 11, extra=2), g["sp_mask_x"])
    np.testing.assert_array_equal(right[:, :-4], left[:, 4:])
    with pytest.raises(ValueError):
        shifted_pair(8, 8, -1)
    with pytest.raises(ValueError):
        shifted_pair(8, 8, 1, cutoff=0.0)


@pytest.mark.parametrize("case,args", [
    ("bm", ("sp_left", "sp_right", 8, 5, "middlebury")),
    ("bm2", ("bm2_left", "bm2_right", 6, 3, "middlebury")),
    ("bm3", ("bm2_right", "bm2_left", 6, 7, "paper")),
    ("bm4", ("bm2_left", "bm2_right", 0, 3, "middlebury")),
])
def test_oracle_baseline_matches_reference(g, case, args):
    lk, rk, d_max, block, sign = args
    d, c, n = O.baseline_bm(g[lk], g[rk], d_max, block, sign=sign)
    np.testing.assert_array_equal(d, g[f"{case}_d"])
    np.testing.assert_allclose(c, g[f"{case}_c"], atol=1e-12, rtol=0)
    assert n == int(g[f"{case}_evals"])


def test_oracle_baseline_validation():
    a = np.zeros((6, 6))
    for bad in [dict(left=a, right=np.zeros((6, 7)), d_max=2, block=3),
                dict(left=a, right=a, d_max=2, block=4),
                dict(left=a, right=a, d_max=2, block=1),
                dict(left=a, right=a, d_max=-1, block=3)]:
        with pytest.raises(ValueError):
            O.baseline_bm(**bad)


def test_oracle_evaluate_matches_reference(g):
    for row in g["ev_reports"]:
        scale = row[0]
        n, bad, s, gi, oi = O.evaluate_counts(g["ev_d"], g["ev_g"], g["ev_inv"], scale)
        assert (n, gi, oi) == (int(row[5]), int(row[6]), int(row[7]))
        for k in range(3):
            assert 100.0 * (bad[k] / n) == row[1 + k]
        assert abs(s / n - row[4]) <= 1e-12


def test_report_text_and_compare():
    from paper_1901_09593_b200.scoring import EvalReport, compare
    r = EvalReport(0.0, 100.0, 0.0, 3.0, 16, 0, 0, total_evals=77, trust_fractions=(0.0, 0.5))
    d = r.to_dict()
    assert d["total_evals"] == 77 and d["trust_fractions"] == [0.0, 0.5]
    text = r.to_text()
    for line in ("bad_2=100.000000", "avg_abs_err=3.000000", "evaluated=16",
                 "trust_fractions=0.000000,0.500000"):
        assert line in text
    assert text.endswith("\n")
    a = EvalReport(1.0, 2.0, 3.0, 0.5, 10, 0, 0, total_evals=300)
    b = EvalReport(1.0, 2.0, 3.0, 0.5, 10, 0, 0, total_evals=1200)
    s = compare(a, b)
    assert all(v == 0.0 for v in s.deltas.values()) and s.eval_ratio == 0.25
    assert compare(EvalReport(1, 1, 1, 1, 1, 0, 0), b).eval_ratio is None
