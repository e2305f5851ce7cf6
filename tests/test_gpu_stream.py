"""Host-output streaming of the C ABI (api.cu launch_streamed): an untimed
mshbm_run_pipeline(MSHBM_IO_HOST) call on a large pair runs level 0's
selection + median in row chunks and copies each chunk's rows to the host
while the next one computes.  The outputs must be bit-identical to the
one-graph path (here: the traced call, which never streams)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,shape", [("C3", (1984, 1056)), ("C2", (1472, 992)),
                                        ("C2", (1101, 611)), ("C4", (1027, 450))])
def test_streamed_outputs_equal_one_graph_outputs(name, shape):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_09593_b200 as gpu
    from paper_1901_09593_b200 import _lib
    from paper_1901_09593_b200.synthetic import CONFIGS, make_pair

    cfg = CONFIGS[name]
    h, w = shape          # >= 1024 rows: the streamed path; odd sizes: partial tiles / chunks
    left, right, _ = make_pair(cfg, height=h, width=w)
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    d_ref, c_ref, trace = gpu.run_pipeline(left, right, mc)       # traced: one graph
    cc = mc.to_c()
    d16 = np.full((h, w), -1, dtype=np.int16)
    c32 = np.full((h, w), np.nan, dtype=np.float32)
    ctx = _lib.context()
    for _ in range(2):                                            # capture, then replay
        d16[:] = -1
        c32[:] = np.nan
        _lib.check(_lib.lib().mshbm_run_pipeline(
            ctx, left.ctypes.data, right.ctypes.data, h, w, w, C.byref(cc), d16.ctypes.data,
            c32.ctypes.data, w, None, None, _lib.IO_HOST, 0, None), ctx)
        assert np.array_equal(d16.astype(np.float64), d_ref)
        assert np.array_equal(c32.astype(np.float64), c_ref)
    # and the traced path still counts every pixel once after streamed runs
    d2, c2, trace2 = gpu.run_pipeline(left, right, mc)
    assert np.array_equal(d2, d_ref) and trace2.total_evals == trace.total_evals
