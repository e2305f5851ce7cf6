"""CPU: pin the C/OpenMP oracle (oracle/mshbm_oracle.c) against the real
reference's outputs (tests/golden, tools/make_golden.py).  It is the oracle
for the configs the reference cannot run in host memory (full C5) and the
CPU baseline of bench.py, so it must reproduce every golden exactly:
disparities and all trace counters equal, costs within 1e-9 (float64
goldens) or the float32 rounding of the stored cost (full-size goldens)."""

import glob
import os

import numpy as np
import pytest

from mshbm_testutil import GOLDEN

CO = pytest.importorskip("oracle.c_oracle")


@pytest.fixture(scope="module", autouse=True)
def _built():
    CO.build()


def test_full_search_matches_reference():
    g = np.load(os.path.join(GOLDEN, "stages.npz"))
    for i in range(24):
        d_max, block, paper = (int(v) for v in g[f"full_p_{i}"])
        d, c = CO.match_coarsest(g[f"full_l_{i}"], g[f"full_r_{i}"], block, d_max,
                                 sign="paper" if paper else "middlebury")
        np.testing.assert_array_equal(d, g[f"full_d_{i}"])
        np.testing.assert_allclose(c, g[f"full_c_{i}"], atol=1e-9, rtol=0)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "pipe_*.npz"))),
                         ids=lambda p: os.path.basename(p)[5:-4])
def test_pipeline_matches_reference(path):
    g = np.load(path)
    d_max, levels, block, radius, paper = (int(v) for v in g["params"])
    alpha, beta = (float(v) for v in g["gates"])
    d, c, counts = CO.run_pipeline(g["left"], g["right"], d_max, levels, block, alpha, beta,
                                   sign="paper" if paper else "middlebury", radius=radius)
    np.testing.assert_array_equal(d, g["disparity"])
    np.testing.assert_allclose(c, g["cost"], atol=1e-9, rtol=0)
    np.testing.assert_array_equal(counts, g["counts"])


@pytest.mark.parametrize("golden", ["full_C2", "full_C4", "full_C3", "crop_C5_2048x1536"])
def test_full_size_matches_reference(golden):
    path = os.path.join(GOLDEN, f"{golden}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
    g = np.load(path)
    cfg = CONFIGS[golden.split("_")[1]]
    if "shape" in g:
        h, w = (int(v) for v in g["shape"])
        left, right, _ = make_pair(cfg, seed=int(g["seed"]), height=h, width=w)
    else:
        left, right, _ = make_pair(cfg, seed=int(g["seed"]))
    d, c, counts = CO.run_pipeline(left, right, cfg.d_max, cfg.levels, cfg.block,
                                   radius=cfg.radius)
    np.testing.assert_array_equal(d, g["disparity"])
    # the golden stores float32 costs: one float32 ulp (at 1.0) of slack
    np.testing.assert_allclose(c, g["cost"].astype(np.float64), atol=1.2e-7, rtol=0)
    np.testing.assert_array_equal(counts, g["counts"])


def test_invalid_arguments_raise():
    x = np.zeros((16, 16))
    with pytest.raises(ValueError):
        CO.run_pipeline(x, x, 64, 5, 5)          # pyramid too deep (pyramid.py:139-151)
    with pytest.raises(ValueError):
        CO.run_pipeline(x, x, 8, 0, 4)           # even block
