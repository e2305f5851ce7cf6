"""CPU: pin the oracle restatement against golden vectors made by the real
reference (tools/make_golden.py).  No GPU needed."""

import glob
import os

import numpy as np
import pytest

from oracle import mshbm_oracle as O

from mshbm_testutil import GOLDEN, counts_of

def _stages():
    return np.load(os.path.join(GOLDEN, "stages.npz"))


def test_downsample_matches_reference():
    g = _stages()
    for i in range(4):
        np.testing.assert_allclose(O.gaussian_downsample(g[f"down_in_{i}"]),
                                   g[f"down_out_{i}"], atol=1e-12, rtol=0)


def test_engine_stats_match_reference():
    g = _stages()
    for i in range(3):
        img = g[f"stats_in_{i}"]
        e = O.Engine(img, img, int(g[f"stats_b_{i}"]), 4)
        np.testing.assert_allclose(e.mean_l, g[f"stats_mean_{i}"], atol=1e-10, rtol=0)
        np.testing.assert_allclose(e.sigma_l, g[f"stats_sigma_{i}"], atol=1e-6, rtol=0)


def test_upsample_bspline_matches_scipy_reference():
    g = _stages()
    for i in range(4):
        h, w = (int(v) for v in g[f"up_shape_{i}"])
        dh, ch = O.upsample_prior(g[f"up_d_{i}"], g[f"up_c_{i}"], (h, w))
        np.testing.assert_array_equal(dh, g[f"up_dhat_{i}"])
        np.testing.assert_allclose(ch, g[f"up_chat_{i}"], atol=1e-13, rtol=0)


def test_selective_median_matches_reference():
    g = _stages()
    for k in range(g["med_d"].shape[0]):
        out = O.selective_median(g["med_d"][k], g["med_c"][k], float(g["med_alpha"][k]))
        np.testing.assert_array_equal(out, g["med_out"][k])


def test_full_search_matches_reference():
    g = _stages()
    for i in range(24):
        d_max, block, paper = (int(v) for v in g[f"full_p_{i}"])
        e = O.Engine(g[f"full_l_{i}"], g[f"full_r_{i}"], block, d_max,
                     sign="paper" if paper else "middlebury")
        d, c = O.match_coarsest(e)
        np.testing.assert_array_equal(d, g[f"full_d_{i}"])
        np.testing.assert_allclose(c, g[f"full_c_{i}"], atol=1e-9, rtol=0)


def test_select_and_refine_match_reference():
    g = _stages()
    e = O.Engine(g["sel_l"], g["sel_r"], 5, 12)
    d, c, st = O.select_with_prior(e, g["sel_dhat"], g["sel_chat"], 0.9, radius=1)
    np.testing.assert_array_equal(d, g["sel_d"])
    np.testing.assert_allclose(c, g["sel_c"], atol=1e-9, rtol=0)
    assert [st["trusted"], st["trusted_evals"], st["window_max"],
            st["full_search_pixels"], st["evals"]] == list(g["sel_stats"])
    e2 = O.Engine(g["sel_l"], g["sel_r"], 5, 12)
    rd, rc = O.refine_level(e2, g["sel_d"], g["sel_c"], 0.9)
    np.testing.assert_array_equal(rd, g["ref_d"])
    np.testing.assert_allclose(rc, g["ref_c"], atol=1e-9, rtol=0)
    assert e2.count == int(g["ref_evals"])


FAST = ["shift64_b11", "paper64_b11", "shift48_k0", "C1_r1", "C1_r2", "C4crop",
        "C2crop"]


@pytest.mark.parametrize("name", FAST)
def test_pipeline_matches_reference(name):
    g = np.load(os.path.join(GOLDEN, f"pipe_{name}.npz"))
    d_max, levels, block, r, paper = (int(v) for v in g["params"])
    alpha, beta = (float(v) for v in g["gates"])
    d, c, tr = O.run_pipeline(g["left"], g["right"], d_max, levels, block,
                              alpha=alpha, beta=beta, radius=r,
                              sign="paper" if paper else "middlebury")
    np.testing.assert_array_equal(d.astype(np.int16), g["disparity"])
    np.testing.assert_allclose(c, g["cost"], atol=1e-9, rtol=0)
    np.testing.assert_array_equal(counts_of(tr), g["counts"])


def test_golden_set_complete():
    names = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "pipe_*.npz")))
    assert len(names) >= 9


def _stage_api():
    return np.load(os.path.join(GOLDEN, "stage_api.npz"))


def test_oracle_plane_volume_matches_reference():
    """CostEngine.plane / full_volume (zncc.py:202-249) incl. the paper sign
    and a flat patch: the oracle's planes equal the reference's volumes."""
    g = _stage_api()
    for i in range(4):
        b, d, paper = (int(v) for v in g[f"vol_p_{i}"])
        e = O.Engine(g[f"vol_l_{i}"], g[f"vol_r_{i}"], b, d,
                     sign="paper" if paper else "middlebury")
        vol = np.stack([e.plane(z) for z in range(d + 1)])
        np.testing.assert_allclose(vol, g[f"vol_{i}"], atol=1e-12, rtol=0)


def test_oracle_dsi_entries_and_slices_match_reference():
    """dsi_entry / dsi_slice / averaged_dsi (zncc.py:304-350) restated on the
    oracle engine's point and row paths."""
    g = _stage_api()
    e = O.Engine(g["pt_l"], g["pt_r"], 3, 4)
    h, w = g["pt_l"].shape
    for k, (i, j, z) in enumerate(g["pt_ijz"]):
        got = e.at(np.array([i]), np.array([j]), np.array([z]))[0]
        assert abs(got - g["pt_entry"][k]) <= 1e-12
        np.testing.assert_allclose(e.dsi_rows(np.array([i]), np.array([j]))[0],
                                   g["pt_slice"][k], atol=1e-12, rtol=0)
        nb = [(i + di, j + dj) for di in (-1, 0, 1) for dj in (-1, 0, 1)
              if 0 <= i + di < h and 0 <= j + dj < w]
        avg = e.dsi_rows(np.array([a for a, _ in nb]), np.array([b for _, b in nb])).sum(0)
        np.testing.assert_allclose(avg, g["pt_avg"][k], atol=1e-12, rtol=0)
    # an empty (all-outside) neighbourhood falls back to the pixel's own row
    np.testing.assert_allclose(e.dsi_rows(np.array([0]), np.array([0]))[0], g["pt_avg_far"],
                               atol=1e-12, rtol=0)


def test_oracle_binomial_smooth_matches_reference():
    g = _stage_api()
    for i in range(3):
        np.testing.assert_allclose(O.binomial_smooth(g[f"bs_in_{i}"]), g[f"bs_out_{i}"],
                                   atol=1e-12, rtol=0)


def test_oracle_match_level_with_prior_matches_reference():
    """match_level_with_prior (matcher.py:362-369) = select -> refine ->
    median, composed from the oracle's stages."""
    g = _stage_api()
    e = O.Engine(g["ml_l"], g["ml_r"], 5, 14)
    d, c, _ = O.select_with_prior(e, g["ml_dhat"], g["ml_chat"], 0.9)
    d, c = O.refine_level(e, d, c, 0.9)
    d = O.selective_median(d, c, 0.9)
    np.testing.assert_array_equal(d, g["ml_d"])
    np.testing.assert_allclose(c, g["ml_c"], atol=1e-12, rtol=0)
