"""Quick device-resident timing of one config through run_pipeline_device."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_09593_b200 as gpu  # noqa: E402
from paper_1901_09593_b200 import _lib  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

import ctypes as C  # noqa: E402
for name in sys.argv[1:] or ["C2"]:
    cfg = CONFIGS[name]
    l, r, _ = make_pair(cfg)
    lt, rt = torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    d, c, tr = gpu.run_pipeline_device(lt, rt, mc, trace=True)
    for _ in range(3):
        gpu.run_pipeline_device(lt, rt, mc, trace=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        gpu.run_pipeline_device(lt, rt, mc, trace=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    # per-stage timing
    gpu.matcher.DIRECT_LAUNCH = False
    _, _, trt = gpu.run_pipeline(l, r, mc)
    print(name, f"{ms:.3f} ms/pair", f"full-search MPD/s {cfg.full_search_pde / ms / 1e3:.0f}",
          f"evaluated {tr.total_evals / ms / 1e3:.0f} MPD/s")
    for lt_ in trt.levels:
        print("   L%d %dx%d d=%d b=%d evals=%d sel=%.3fms med=%.3fms up=%.3fms" % (
            lt_.level, lt_.width, lt_.height, lt_.d_max, lt_.block, lt_.evals,
            lt_.seconds["select"] * 1e3, lt_.seconds["median"] * 1e3,
            lt_.seconds.get("upsample", 0) * 1e3))
tf, ms = C.c_double(), C.c_double()
_lib.lib().mshbm_probe_fp32_peak(0, 20000, C.byref(tf), C.byref(ms))
print(f"fp32 FFMA probe: {tf.value:.1f} TFLOP/s ({ms.value:.2f} ms)")
_lib.lib().mshbm_probe_fp64_peak(0, 4000, C.byref(tf), C.byref(ms))
print(f"fp64 DFMA probe: {tf.value:.1f} TFLOP/s ({ms.value:.2f} ms)")
