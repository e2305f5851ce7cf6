"""C4 batch throughput vs the number of slot streams of mshbm_run_batch
(measurement helper: python tools/c4_streams.py on a B200)."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_1901_09593_b200 as gpu
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
cfg = CONFIGS["C4"]
imgs = [make_pair(cfg, seed=cfg.seed + i) for i in range(cfg.batch)]
L = torch.stack([torch.from_numpy(x[0]) for x in imgs]).cuda()
R = torch.stack([torch.from_numpy(x[1]) for x in imgs]).cuda()
mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
for ns in (2, 4, 6, 8, 4):
    for _ in range(3): gpu.run_batch(L, R, mc, n_streams=ns, trace=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): gpu.run_batch(L, R, mc, n_streams=ns, trace=False)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(ns, f"{ms:.2f} ms/batch", f"{cfg.batch / ms * 1e3:.0f} pairs/s")
