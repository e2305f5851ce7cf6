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
