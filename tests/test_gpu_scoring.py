"""GPU: the §8(f) "next" rows through the drop-in API -- ``baseline_bm``
(fused full-search sweep) and ``evaluate`` (device reduction) -- against the
reference's golden vectors and the oracle.  Mirrors the semantics of the
reference's tests/test_baseline_eval.py.

Tolerances: baseline disparities bit-exact (the goldens hold no near-ties),
costs within 1e-4 (BASELINE north_star; observed ~1e-6); evaluate counts
exact, rates bit-identical, mean absolute error within 1e-12 relative
(device fp64 sum order differs from numpy's pairwise sum).
"""

import os

import numpy as np
import pytest

from oracle import mshbm_oracle as O

from mshbm_testutil import GOLDEN

pytestmark = pytest.mark.gpu
COST_TOL = 1e-4


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_09593_b200 as g
    return g


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "scoring.npz"))


def _gt(g, values, invalid=None):
    values = np.asarray(values, dtype=np.float64).copy()
    invalid = np.zeros(values.shape, bool) if invalid is None else invalid
    values[invalid] = np.nan
    return g.GroundTruthDisparity(values=values, invalid=invalid)


@pytest.mark.parametrize("case,args", [
    ("bm", ("sp_left", "sp_right", 8, 5, "middlebury")),
    ("bm2", ("bm2_left", "bm2_right", 6, 3, "middlebury")),
    ("bm3", ("bm2_right", "bm2_left", 6, 7, "paper")),
    ("bm4", ("bm2_left", "bm2_right", 0, 3, "middlebury")),
])
def test_baseline_matches_reference_golden(gpu, gold, case, args):
    lk, rk, d_max, block, sign = args
    d, c, n = gpu.baseline_bm(gold[lk], gold[rk], d_max, block, sign=sign)
    np.testing.assert_array_equal(d, gold[f"{case}_d"])
    np.testing.assert_allclose(c, gold[f"{case}_c"], atol=COST_TOL, rtol=0)
    assert n == int(gold[f"{case}_evals"])


def test_baseline_identical_pair(gpu):
    img = np.random.default_rng(1).random((10, 14))
    d, c, n = gpu.baseline_bm(img, img, 5, 3)
    assert np.all(d[1:-1, 1:-1] == 0)
    assert n == 10 * 14 * 6


def test_baseline_eval_count_closed_form(gpu):
    rng = np.random.default_rng(2)
    for h, w, d_max in [(7, 9, 0), (12, 31, 4), (33, 20, 17)]:
        left, right = rng.random((h, w)), rng.random((h, w))
        _, _, n = gpu.baseline_bm(left, right, d_max, 3)
        assert n == h * w * (d_max + 1)


def test_baseline_recovers_constant_shift(gpu):
    left, right = gpu.shifted_pair(24, 40, 4, np.random.default_rng(3), cutoff=0.15)
    d, _, _ = gpu.baseline_bm(left, right, 8, 5)
    mask = gpu.interior_mask(left.shape, 4, 5)
    assert np.mean(d[mask] == 4) >= 0.95


@pytest.mark.parametrize("seed,h,w,d_max,block,sign", [
    (10, 40, 64, 24, 9, "middlebury"), (11, 37, 53, 13, 11, "paper"),
    (12, 64, 96, 40, 5, "middlebury"), (13, 30, 30, 29, 15, "middlebury"),
])
def test_baseline_matches_oracle_random(gpu, seed, h, w, d_max, block, sign):
    rng = np.random.default_rng(seed)
    left, right = gpu.shifted_pair(h, w, 5, rng, cutoff=0.2)
    if sign == "paper":
        left, right = right, left
    right = right + 1e-3 * rng.standard_normal(right.shape)
    d, c, n = gpu.baseline_bm(left, right, d_max, block, sign=sign)
    od, oc, on = O.baseline_bm(left, right, d_max, block, sign=sign)
    assert n == on
    agree = d == od
    assert agree.mean() >= 1 - 5e-4
    assert np.abs(c - oc)[agree].max() <= COST_TOL


def test_baseline_validation(gpu):
    a = np.zeros((8, 8))
    with pytest.raises(ValueError):
        gpu.baseline_bm(a, np.zeros((8, 9)), 2, 3)
    with pytest.raises(ValueError):
        gpu.baseline_bm(a, a, 2, 4)
    with pytest.raises(ValueError):
        gpu.baseline_bm(a, a, -1, 3)
    with pytest.raises(ValueError):
        gpu.baseline_bm(a, a, 2, 3, sign="bogus")


def test_evaluate_matches_reference_golden(gpu, gold):
    gt = gpu.GroundTruthDisparity(values=gold["ev_g"], invalid=gold["ev_inv"])
    for row in gold["ev_reports"]:
        r = gpu.evaluate(gold["ev_d"], gt, scale=float(row[0]))
        assert (r.evaluated, r.gt_invalid, r.output_invalid) == tuple(int(v) for v in row[5:8])
        assert (r.bad_1, r.bad_2, r.bad_4) == (row[1], row[2], row[3])
        assert abs(r.avg_abs_err - row[4]) <= 1e-12 * max(1.0, row[4])


def test_evaluate_exact_and_offset(gpu):
    v = np.arange(64, dtype=np.float64).reshape(8, 8)
    r = gpu.evaluate(v, _gt(gpu, v))
    assert (r.bad_2, r.avg_abs_err, r.evaluated) == (0.0, 0.0, 64)
    r = gpu.evaluate(v + 3.0, _gt(gpu, v))
    assert (r.bad_1, r.bad_2, r.bad_4, r.avg_abs_err) == (100.0, 100.0, 0.0, 3.0)


def test_evaluate_matches_counting_oracle(gpu):
    rng = np.random.default_rng(4)
    for _ in range(10):
        gv = rng.uniform(0, 40, size=(9, 11))
        inv = rng.random((9, 11)) < 0.15
        d = gv + rng.normal(0, 2.5, size=(9, 11))
        d[rng.random((9, 11)) < 0.1] = np.nan
        r = gpu.evaluate(d, _gt(gpu, gv, inv))
        n, bad, s, gi, oi = O.evaluate_counts(d, gv, inv)
        assert (r.evaluated, r.gt_invalid, r.output_invalid) == (n, gi, oi)
        for k, v in enumerate((r.bad_1, r.bad_2, r.bad_4)):
            assert abs(v - 100.0 * bad[k] / n) <= 1e-9
        assert abs(r.avg_abs_err - s / n) <= 1e-9


def test_evaluate_scale_sign_and_errors(gpu):
    gv = np.full((6, 6), 8.0)
    assert gpu.evaluate(np.full((6, 6), 2.0), _gt(gpu, gv), scale=4.0).avg_abs_err == 0.0
    r = gpu.evaluate(np.full((6, 6), 1.0), _gt(gpu, gv), scale=4.0)
    assert r.avg_abs_err == 4.0 and r.bad_2 == 100.0
    rng = np.random.default_rng(5)
    gv = rng.uniform(5, 20, (7, 7))
    e = rng.uniform(0, 6, (7, 7))
    p, m = gpu.evaluate(gv + e, _gt(gpu, gv)), gpu.evaluate(gv - e, _gt(gpu, gv))
    assert (p.bad_1, p.bad_2, p.bad_4) == (m.bad_1, m.bad_2, m.bad_4)
    assert abs(p.avg_abs_err - m.avg_abs_err) <= 1e-9
    with pytest.raises(ValueError):
        gpu.evaluate(np.zeros((4, 5)), _gt(gpu, np.zeros((5, 4))))
    with pytest.raises(ValueError):
        gpu.evaluate(np.zeros((4, 4)), _gt(gpu, np.zeros((4, 4))), scale=0.0)
    # every pixel invalid: zero rates, nothing evaluated
    r = gpu.evaluate(np.full((3, 3), np.nan), _gt(gpu, np.zeros((3, 3))))
    assert (r.evaluated, r.output_invalid, r.bad_1, r.avg_abs_err) == (0, 9, 0.0, 0.0)


def test_evaluate_device_tensor_large(gpu):
    """Full-size map already in HBM (no host copy of the disparity)."""
    import torch
    h, w = 1984, 2944
    rng = np.random.default_rng(6)
    d = rng.uniform(0, 200, (h, w))
    d[rng.random((h, w)) < 0.01] = np.nan
    gv = d + rng.normal(0, 2, (h, w))
    inv = rng.random((h, w)) < 0.05
    r = gpu.evaluate(torch.from_numpy(d).cuda(), _gt(gpu, gv, inv))
    n, bad, s, gi, oi = O.evaluate_counts(d, gv, inv)
    assert (r.evaluated, r.gt_invalid, r.output_invalid) == (n, gi, oi)
    assert r.bad_1 == 100.0 * (bad[0] / n)
    assert abs(r.avg_abs_err - s / n) <= 1e-12 * (s / n)


def test_hierarchy_vs_baseline_on_easy_pairs(gpu):
    rng = np.random.default_rng(6)
    for shift in (3, 7):
        left, right = gpu.shifted_pair(64, 80, shift, rng, cutoff=0.04)
        mask = gpu.interior_mask(left.shape, shift, 11, extra=2)
        gt = _gt(gpu, np.full(left.shape, float(shift)), ~mask)
        d, _, trace = gpu.run_pipeline(left, right, gpu.MatchConfig(d_max=16, levels=2, block=11))
        bd, _, bn = gpu.baseline_bm(left, right, 16, 11)
        ours, base = gpu.evaluate(d, gt), gpu.evaluate(bd, gt)
        assert ours.avg_abs_err <= base.avg_abs_err + 0.1
        assert trace.total_evals < bn
    left, right = gpu.shifted_pair(128, 128, 5, np.random.default_rng(7), cutoff=0.02)
    gt = _gt(gpu, np.full(left.shape, 5.0), ~gpu.interior_mask(left.shape, 5, 11, extra=2))
    d, _, trace = gpu.run_pipeline(left, right, gpu.MatchConfig(d_max=32, levels=2, block=11))
    ours = gpu.evaluate(d, gt)
    ours.total_evals = trace.total_evals
    bd, _, bn = gpu.baseline_bm(left, right, 32, 11)
    base = gpu.evaluate(bd, gt)
    base.total_evals = bn
    assert bn == 128 * 128 * 33
    s = gpu.compare(ours, base)
    assert s.eval_ratio is not None and s.eval_ratio < 0.25
    assert s.deltas["avg_abs_err"] <= 0.1


# ---------------------------------------------------------------- codecs
def test_pnm_device_upload_matches_host_decode(gpu, gold, tmp_path):
    import torch
    g = np.load(os.path.join(GOLDEN, "formats.npz"))
    for name in ("p5", "p6_16", "p6_8", "pgm16", "p2"):
        p = tmp_path / name
        p.write_bytes(bytes(g[f"file_{name}"]))
        dev = gpu.load_pnm_device(p)
        assert dev.is_cuda and dev.dtype == torch.float32
        ref = g[f"dec_{name}"].astype(np.float32)
        np.testing.assert_allclose(dev.cpu().numpy(), ref, rtol=0, atol=1e-7)
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n2 2\n100\n" + bytes([0, 50, 100, 255]))
    with pytest.raises(gpu.DecodeError):
        gpu.load_pnm_device(bad)


def test_pipeline_from_pgm_files(gpu, tmp_path):
    """File -> device decode -> pipeline -> PFM, against the host-array path."""
    left, right = gpu.shifted_pair(96, 128, 6, np.random.default_rng(8), cutoff=0.1)
    gpu.write_pgm(left, tmp_path / "l.pgm", maxval=65535)
    gpu.write_pgm(right, tmp_path / "r.pgm", maxval=65535)
    cfg = gpu.MatchConfig(d_max=16, levels=2, block=5)
    lh, rh = gpu.read_pnm(tmp_path / "l.pgm"), gpu.read_pnm(tmp_path / "r.pgm")
    d_host, c_host, _ = gpu.run_pipeline(lh, rh, cfg)
    ld, rd = gpu.load_pnm_device(tmp_path / "l.pgm"), gpu.load_pnm_device(tmp_path / "r.pgm")
    d_dev, c_dev, _ = gpu.run_pipeline_device(ld, rd, cfg)
    np.testing.assert_array_equal(d_dev.cpu().numpy().astype(np.float64), d_host)
    np.testing.assert_array_equal(c_dev.cpu().numpy().astype(np.float64), c_host)
    gpu.write_disparity_pfm(d_dev, tmp_path / "d.pfm")
    back = gpu.read_pfm(tmp_path / "d.pfm")
    np.testing.assert_array_equal(back.values, d_host)
