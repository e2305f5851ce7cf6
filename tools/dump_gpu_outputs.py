"""Run every golden pipeline case on the GPU and save outputs for offline
analysis (gpurun_out/dump_<name>.npz)."""
import glob
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1901_09593_b200 as gpu  # noqa: E402
from mshbm_testutil import counts_of  # noqa: E402

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for p in sorted(glob.glob(os.path.join(ROOT, "tests/golden/pipe_*.npz"))):
    g = np.load(p)
    name = os.path.basename(p)[5:-4]
    d_max, levels, block, r, paper = (int(v) for v in g["params"])
    cfg = gpu.MatchConfig(d_max=d_max, levels=levels, block=block, radius=r,
                          sign="paper" if paper else "middlebury")
    d, c, tr = gpu.run_pipeline(g["left"], g["right"], cfg)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"dump_{name}.npz"), d=d, c=c,
                        counts=counts_of(tr))
    same = d == g["disparity"]
    print(name, "mism", int((~same).sum()), "cerr", float(np.abs(c - g["cost"])[same].max()),
          "n_cerr>1e-4", int((np.abs(c - g["cost"]) > 1e-4)[same].sum()))
