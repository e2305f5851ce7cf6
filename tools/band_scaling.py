"""C5 row-band sharding on one B200: time every band of a world-N split
(mshbm_run_pipeline_band, device IO, CUDA events) and compare the slowest band
with the whole-image pipeline.  T(N) >= max band time (+ the NCCL gather of the
bands, not included), so whole / (N * max band) bounds the scaling efficiency
the band decomposition allows (halo rows and redundant coarse-level work).
    python tools/band_scaling.py [C5] [2 4 8]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
worlds = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
cfg = CONFIGS[name]
left, right, _ = make_pair(cfg)
L, R = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


whole = timed(lambda: gpu.run_pipeline_device(L, R, mc, trace=False))
print(f"{name} whole image: {whole:.2f} ms")
for n in worlds:
    bands = gpu.sharding.plan_bands(cfg.height, n, cfg.levels)
    ts = [timed(lambda b=b: gpu.run_pipeline_band(L, R, mc, b[0], b[1], trace=False))
          for b in bands]
    print(f"world {n}: band ms {[round(t, 2) for t in ts]}  max {max(ts):.2f}  "
          f"efficiency bound {whole / (n * max(ts)):.3f}")
