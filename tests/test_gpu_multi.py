"""GPU: the C4 batch API and the C5 row-band decomposition on one device.

Bands are emulated sequentially on one GPU (the multi-rank path only adds a
gather): every band must reproduce its rows of the whole-image run
bit-for-bit, and the per-band traces must sum to the whole-image trace."""

import numpy as np
import pytest

from mshbm_testutil import counts_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_09593_b200 as g
    return g


@pytest.mark.parametrize("name,shape,world", [("C5", (384, 512), 3), ("C2", (248, 368), 2),
                                              ("C3", (256, 320), 4), ("C1", (375, 450), 3)])
def test_row_bands_reproduce_whole_image(gpu, name, shape, world):
    import torch
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
    cfg = CONFIGS[name]
    left, right, _ = make_pair(cfg, seed=cfg.seed + 5, height=shape[0], width=shape[1])
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    d, c, tr = gpu.run_pipeline_device(lt, rt, mc)
    bands = gpu.sharding.plan_bands(shape[0], world, cfg.levels)
    parts_d, parts_c, traces = [], [], []
    for b0, b1 in bands:
        bd, bc, bt = gpu.run_pipeline_band(lt, rt, mc, b0, b1)
        parts_d.append(bd)
        parts_c.append(bc)
        traces.append(bt)
    assert torch.equal(torch.cat(parts_d), d)
    assert torch.equal(torch.cat(parts_c), c)
    merged = gpu.sharding.merge_traces(traces)
    np.testing.assert_array_equal(counts_of(merged), counts_of(tr))


def test_row_band_limits_validated(gpu):
    import torch
    x = torch.rand(64, 64, device="cuda") * 255
    mc = gpu.MatchConfig(d_max=16, levels=2, block=5)
    with pytest.raises(ValueError):
        gpu.run_pipeline_band(x, x, mc, 2, 32)      # not a multiple of 4
    with pytest.raises(ValueError):
        gpu.run_pipeline_band(x, x, mc, 32, 16)


def test_batch_matches_single_pair_runs(gpu):
    import torch
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
    cfg = CONFIGS["C4"]
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    pairs = [make_pair(cfg, seed=cfg.seed + i, height=180, width=320) for i in range(6)]
    L = torch.stack([torch.from_numpy(p[0]) for p in pairs]).cuda()
    R = torch.stack([torch.from_numpy(p[1]) for p in pairs]).cuda()
    D, Cc, traces = gpu.run_batch(L, R, mc, n_streams=3)
    torch.cuda.synchronize()
    for i in range(6):
        d, c, t = gpu.run_pipeline_device(L[i], R[i], mc)
        assert torch.equal(D[i], d) and torch.equal(Cc[i], c)
        assert traces[i].counts_dict() == t.counts_dict()


def test_row_bands_on_smooth_low_contrast_pair(gpu):
    """The reference's constant-shift fixture (smooth, [0, 1]): under
    MSHBM_SWEEP4=2 sweep4's precision guard flags tiles of it, so bands also
    exercise the sweep2 fixup job list (test_gpu_sweep4 runs this file with
    the override); either way bands must reproduce the whole image."""
    import torch
    from mshbm_testutil import load_golden
    g = load_golden("pipe_shift48_k0.npz")
    d_max, levels, block, r, _ = (int(v) for v in g["params"])
    mc = gpu.MatchConfig(d_max=d_max, levels=levels, block=block, radius=r)
    lt = torch.from_numpy(np.ascontiguousarray(g["left"], dtype=np.float32)).cuda()
    rt = torch.from_numpy(np.ascontiguousarray(g["right"], dtype=np.float32)).cuda()
    d, c, tr = gpu.run_pipeline_device(lt, rt, mc)
    h = lt.shape[0]
    bands = gpu.sharding.plan_bands(h, 2, levels)
    parts_d, parts_c, traces = [], [], []
    for b0, b1 in bands:
        bd, bc, bt = gpu.run_pipeline_band(lt, rt, mc, b0, b1)
        parts_d.append(bd)
        parts_c.append(bc)
        traces.append(bt)
    assert torch.equal(torch.cat(parts_d), d)
    assert torch.equal(torch.cat(parts_c), c)
    np.testing.assert_array_equal(counts_of(gpu.sharding.merge_traces(traces)), counts_of(tr))
