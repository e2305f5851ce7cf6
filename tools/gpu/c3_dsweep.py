"""C3 images at several d_max: level-0 selection time (timed graph replay)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
cfg = CONFIGS["C3"]
l, r, _ = make_pair(cfg)
gpu.matcher.DIRECT_LAUNCH = False
for d in [int(x) for x in sys.argv[1:]] or [255, 256, 287, 288]:
    mc = gpu.MatchConfig(d_max=d, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    best = 1e9
    for _ in range(4):
        _, _, t = gpu.run_pipeline(l, r, mc)
        best = min(best, t.levels[-1].seconds["select"] * 1e3)
    print("d_max", d, "L0 select %.3f ms" % best, flush=True)
