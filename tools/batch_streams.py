"""C4 batch throughput vs the number of slot streams (mshbm_run_batch):
    python tools/batch_streams.py [2 4 8 16]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

cfg = CONFIGS["C4"]
imgs = [make_pair(cfg, seed=cfg.seed + i) for i in range(cfg.batch)]
L = torch.stack([torch.from_numpy(x[0]) for x in imgs]).cuda()
R = torch.stack([torch.from_numpy(x[1]) for x in imgs]).cuda()
mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
for ns in [int(x) for x in sys.argv[1:]] or [2, 4, 8, 16]:
    for _ in range(2):
        gpu.run_batch(L, R, mc, n_streams=ns, trace=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gpu.run_batch(L, R, mc, n_streams=ns, trace=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"streams {ns}: {ms:.2f} ms per 64-pair batch, {cfg.batch / ms * 1e3:.0f} pairs/s")
