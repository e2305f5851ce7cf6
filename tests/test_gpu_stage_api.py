"""Stage APIs off run_pipeline's path against the real reference
(tests/golden/stage_api.npz, tools/make_golden.py stage_api):

* CostEngine.plane / full_volume (zncc.py:202-249), incl. the paper sign and
  a flat (sigma < eps) patch, and the EvalCounter tally (zncc.py:85-102);
* dsi_entry, dsi_slice, averaged_dsi incl. corner clipping and the
  empty-neighbourhood fallback (zncc.py:304-350);
* match_level_with_prior (matcher.py:362-369);
* binomial_smooth (pyramid.py:65-68).

The engine's point/plane/row paths are fp64 like the reference, so costs
match to 1e-9 (the reference tests' own tolerance, tests/test_zncc.py).
"""

import numpy as np
import pytest

from mshbm_testutil import load_golden, parity_report

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_09593_b200 as g
    return g


@pytest.fixture(scope="module")
def gold():
    return load_golden("stage_api.npz")


@pytest.mark.parametrize("i", range(4))
def test_plane_and_full_volume_match_reference(gpu, gold, i):
    b, d, paper = (int(v) for v in gold[f"vol_p_{i}"])
    sign = "paper" if paper else "middlebury"
    e = gpu.CostEngine(gold[f"vol_l_{i}"], gold[f"vol_r_{i}"], block=b, d_max=d, sign=sign)
    vol = e.full_volume()
    ref = gold[f"vol_{i}"]
    assert vol.shape == ref.shape == (d + 1,) + gold[f"vol_l_{i}"].shape
    np.testing.assert_allclose(vol, ref, atol=1e-9, rtol=0)
    assert e.counter.count == int(gold[f"vol_count_{i}"])
    assert vol.min() >= -1.0 and vol.max() <= 1.0
    # one plane on its own equals the volume's slice; the count adds H*W
    z = d // 2
    np.testing.assert_array_equal(e.plane(z), vol[z])
    assert e.counter.count == int(gold[f"vol_count_{i}"]) + vol[0].size


def test_dsi_entry_slice_and_averaged_dsi_match_reference(gpu, gold):
    e = gpu.CostEngine(gold["pt_l"], gold["pt_r"], block=3, d_max=4)
    for k, (i, j, z) in enumerate(gold["pt_ijz"]):
        assert abs(gpu.dsi_entry(e, int(i), int(j), int(z)) - gold["pt_entry"][k]) <= 1e-9
    for k, (i, j, _) in enumerate(gold["pt_ijz"]):
        s = e.dsi_slice(int(i), int(j))
        assert s.pixel == (int(i), int(j))
        np.testing.assert_allclose(s.costs, gold["pt_slice"][k], atol=1e-9, rtol=0)
    for k, (i, j, _) in enumerate(gold["pt_ijz"]):
        a = gpu.averaged_dsi(e, int(i), int(j))
        np.testing.assert_allclose(a.costs, gold["pt_avg"][k], atol=1e-9, rtol=0)
    far = [(-5, -5), (-6, 0), (0, -9)]
    np.testing.assert_allclose(gpu.averaged_dsi(e, 0, 0, neighborhood=far).costs,
                               gold["pt_avg_far"], atol=1e-9, rtol=0)
    # the same sequence of calls tallies the same evaluations
    assert e.counter.count == int(gold["pt_count"])


def test_dsi_entry_rejects_out_of_range_z(gpu, gold):
    e = gpu.CostEngine(gold["pt_l"], gold["pt_r"], block=3, d_max=4)
    with pytest.raises(ValueError):
        gpu.dsi_entry(e, 1, 1, 5)
    with pytest.raises(ValueError):
        gpu.dsi_entry(e, 1, 1, -1)


def test_match_level_with_prior_matches_reference(gpu, gold):
    e = gpu.CostEngine(gold["ml_l"], gold["ml_r"], block=5, d_max=14)
    d, c = gpu.match_level_with_prior(e, gold["ml_dhat"], gold["ml_chat"], 0.9, 0.9)
    assert d.dtype == np.float64 and c.dtype == np.float64
    frac, cerr, _ = parity_report(d, c, gold["ml_d"], gold["ml_c"])
    assert frac == 0.0
    assert cerr <= 1e-5     # the selection/refine sweeps score in fp32 (DESIGN 4)
    assert e.counter.count == int(gold["ml_count"])


@pytest.mark.parametrize("i", range(3))
def test_binomial_smooth_matches_reference(gpu, gold, i):
    from paper_1901_09593_b200.pyramid import binomial_smooth
    out = binomial_smooth(gold[f"bs_in_{i}"])
    np.testing.assert_allclose(out, gold[f"bs_out_{i}"], atol=1e-10, rtol=0)
