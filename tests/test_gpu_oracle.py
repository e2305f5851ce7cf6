"""GPU vs the CPU oracle on seeded random cases: odd sizes, both sign
conventions, K = 0 (single level), radii 0-3, blocks 3-13 (incl. the
generic fallback kernel), narrow images (width < d_max), plus the
BASELINE generator at parity size for every config."""

import numpy as np
import pytest

from mshbm_testutil import counts_close, counts_of, parity_report

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_09593_b200 as g
    return g


CASES = [
    # (h, w, d_max, levels, block, radius, sign, seed)
    (37, 53, 12, 0, 3, 1, "middlebury", 1),
    (64, 64, 16, 2, 11, 1, "middlebury", 2),
    (64, 80, 16, 2, 11, 2, "paper", 3),
    (96, 70, 24, 1, 5, 0, "middlebury", 4),
    (81, 123, 32, 2, 7, 3, "paper", 5),
    (50, 40, 60, 1, 9, 2, "middlebury", 6),     # width < d_max
    (60, 90, 20, 1, 13, 1, "middlebury", 7),    # generic fallback kernel
    (128, 160, 16, 2, 7, 1, "middlebury", 8),
    (72, 96, 24, 1, 7, 5, "paper", 9),          # radius 5: the 15-wide trusted-window path
    (88, 100, 40, 2, 9, 4, "middlebury", 10),
    (61, 77, 16, 1, 5, 2, "middlebury", 11),    # odd height: a lone last pixel row
]


def _pair(h, w, seed):
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
    left, right, _ = make_pair(CONFIGS["C4"], seed=seed, height=h, width=w)
    return left, right


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}-D{c[2]}-K{c[3]}-b{c[4]}-r{c[5]}-{c[6]}"
                                             for c in CASES])
def test_random_cases_match_oracle(gpu, case):
    from oracle import mshbm_oracle as O
    h, w, d_max, levels, block, radius, sign, seed = case
    left, right = _pair(h, w, seed)
    cfg = gpu.MatchConfig(d_max=d_max, levels=levels, block=block, radius=radius, sign=sign)
    d, c, tr = gpu.run_pipeline(left, right, cfg)
    od, oc, otr = O.run_pipeline(left, right, d_max, levels, block, radius=radius, sign=sign)
    frac, cerr, med = parity_report(d, c, od, oc)
    assert frac <= 5e-4 or (frac * d.size) <= 1, f"{frac:.4%} flipped"
    assert cerr <= 1e-4 and med <= 1e-6
    assert counts_close(counts_of(tr), counts_of(otr))


def test_uniform_images_are_degenerate(gpu):
    """Flat blocks (sigma < sigma_eps) cost -1 everywhere: disparity 0."""
    flat = np.full((40, 48), 77.0, dtype=np.float32)
    cfg = gpu.MatchConfig(d_max=8, levels=1, block=5, radius=1)
    d, c, tr = gpu.run_pipeline(flat, flat, cfg)
    assert np.all(c <= -1.0 + 1e-12) and np.all(c >= -1.0 - 1e-12)
    assert np.all(d == 0)


def test_identical_pair_gives_zero_disparity(gpu):
    left, _ = _pair(48, 64, 9)
    cfg = gpu.MatchConfig(d_max=16, levels=2, block=5)
    d, c, _ = gpu.run_pipeline(left, left, cfg)
    inner = np.s_[3:-3, 3:-3]
    assert np.mean(d[inner] == 0) >= 0.99
    assert np.all(c <= 1.0) and np.all(c >= -1.0)


def test_user_pyramid_matches_built_pyramid(gpu):
    left, right = _pair(64, 96, 10)
    cfg = gpu.MatchConfig(d_max=24, levels=2, block=5, radius=2)
    pyr = gpu.build_pyramid(left, right, 24, levels=2, base_block=5)
    d1, c1, t1 = gpu.run_pipeline(left, right, cfg)
    d2, c2, t2 = gpu.run_pipeline(None, None, cfg, pyramid=pyr)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_allclose(c1, c2, atol=1e-6)
    assert t1.counts_dict() == t2.counts_dict()


@pytest.mark.parametrize("name,shape", [("C1", (120, 160)), ("C2", (176, 272)),
                                        ("C3", (192, 320)), ("C4", (136, 240)),
                                        ("C5", (192, 256))])
def test_baseline_configs_at_parity_size(gpu, name, shape):
    from oracle import mshbm_oracle as O
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
    cfg = CONFIGS[name]
    left, right, _ = make_pair(cfg, seed=cfg.seed + 77, height=shape[0], width=shape[1])
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    d, c, tr = gpu.run_pipeline(left, right, mc)
    od, oc, otr = O.run_pipeline(left, right, cfg.d_max, cfg.levels, cfg.block,
                                 radius=cfg.radius)
    frac, cerr, med = parity_report(d, c, od, oc)
    assert frac <= 5e-4 or (frac * d.size) <= 2, f"{name}: {frac:.4%} flipped"
    assert cerr <= 1e-4 and med <= 1e-6
    assert counts_close(counts_of(tr), counts_of(otr))


def test_gate_variants_match_oracle(gpu):
    """Non-default alpha/beta move many pixels across the gates."""
    from oracle import mshbm_oracle as O
    left, right = _pair(96, 128, 21)
    for alpha, beta in ((0.5, 0.99), (0.97, 0.6)):
        cfg = gpu.MatchConfig(d_max=24, levels=2, block=5, radius=2, alpha=alpha, beta=beta)
        d, c, tr = gpu.run_pipeline(left, right, cfg)
        od, oc, otr = O.run_pipeline(left, right, 24, 2, 5, alpha=alpha, beta=beta, radius=2)
        frac, cerr, med = parity_report(d, c, od, oc)
        assert frac <= 5e-4 or frac * d.size <= 2
        assert cerr <= 1e-4 and med <= 1e-6
        assert counts_close(counts_of(tr), counts_of(otr))


def test_unit_range_images_match_oracle(gpu):
    """[0, 1] float64 images (the reference test-suite convention)."""
    from oracle import mshbm_oracle as O
    rng = np.random.default_rng(33)
    left = rng.random((40, 56))
    right = np.roll(left, -3, axis=1) + 0.01 * rng.random((40, 56))
    cfg = gpu.MatchConfig(d_max=8, levels=1, block=5)
    d, c, _ = gpu.run_pipeline(left, right, cfg)
    od, oc, _ = O.run_pipeline(left, right, 8, 1, 5)
    frac, cerr, med = parity_report(d, c, od, oc)
    assert frac <= 1e-3 and cerr <= 1e-4


def test_tiny_and_degenerate_shapes(gpu):
    from oracle import mshbm_oracle as O
    rng = np.random.default_rng(34)
    for h, w in ((3, 3), (4, 7), (9, 2)):
        left, right = rng.random((h, w)) * 255, rng.random((h, w)) * 255
        cfg = gpu.MatchConfig(d_max=3, levels=0, block=3)
        d, c, _ = gpu.run_pipeline(left, right, cfg)
        od, oc, _ = O.run_pipeline(left, right, 3, 0, 3)
        np.testing.assert_array_equal(d, od)
        np.testing.assert_allclose(c, oc, atol=1e-5)
    with pytest.raises(ValueError):
        gpu.run_pipeline(np.zeros((0, 5)), np.zeros((0, 5)), gpu.MatchConfig(d_max=2, levels=0))
    with pytest.raises(ValueError):
        gpu.run_pipeline(np.zeros((8, 8)), np.zeros((8, 9)), gpu.MatchConfig(d_max=4, levels=0))
    with pytest.raises(ValueError):   # too deep (pyramid.py:139-151)
        gpu.run_pipeline(np.zeros((16, 16)), np.zeros((16, 16)), gpu.MatchConfig(d_max=64, levels=3))
