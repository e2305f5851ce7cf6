"""Per-level stage times of one C5 row band (world N, band index i) next to
the whole-image run (timed graph replay, CUDA events):
    python tools/band_stages.py [N] [i]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
bi = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS["C5"]
left, right, _ = make_pair(cfg)
L, R = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
b0, b1 = gpu.sharding.plan_bands(cfg.height, n, cfg.levels)[bi]


def stages(tr):
    return [(lt.level, lt.seconds["select"] * 1e3, lt.seconds["median"] * 1e3,
             lt.seconds.get("upsample", 0.0) * 1e3) for lt in tr.levels]


for _ in range(2):
    _, _, tw = gpu.run_pipeline_device(L, R, mc, trace=True)
    _, _, tb = gpu.run_pipeline_band(L, R, mc, b0, b1, trace=True, timed=True)
print(f"band {bi} of {n}: rows [{b0}, {b1})  build whole {tw.build_seconds * 1e3:.3f} ms, "
      f"band {tb.build_seconds * 1e3:.3f} ms")
for (k, s, m, u), (_, sb, mb, ub) in zip(stages(tw), stages(tb)):
    print(f"  L{k}: whole/{n} sel {s / n:.3f} med {m / n:.3f} up {u / n:.3f} | band sel {sb:.3f} "
          f"med {mb:.3f} up {ub:.3f}")
