"""One direct-launch pipeline run of a config (for ncu): python tools/prof_once.py C2"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
l, r, _ = make_pair(cfg)
gpu.matcher.DIRECT_LAUNCH = False
d, c, t = gpu.run_pipeline(l, r, gpu.MatchConfig(d_max=int(os.environ.get("MSHBM_DMAX", cfg.d_max)), levels=cfg.levels,
                                                 block=cfg.block, radius=cfg.radius))
print(cfg.name, "ok", t.total_evals, [round(lv.seconds["select"] * 1e3, 3) for lv in t.levels])
