"""Explain level-0 disparity mismatches of one full-size golden (GPU box).

    python tools/diag_mismatch.py oracle_C5 [direct|graph]

For every mismatch that is neither a near tie nor a 5x5-median descendant of
one, print the reference-side quantities that decide the pixel: the prior
(d_hat, c_hat from the C oracle's level-1 maps, i.e. the reference's), the
trusted gate margin c_hat - beta, the selection cost C_sel and its margin to
alpha, the best two candidates of the selection and of the 3x3-summed
refinement with their gaps, and the GPU's teacher-forced level-0 answer.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402

import paper_1901_09593_b200 as gpu  # noqa: E402
from mshbm_testutil import classify_mismatches  # noqa: E402
from oracle import c_oracle as CO  # noqa: E402
from oracle import mshbm_oracle as O  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402


def main():
    name = sys.argv[1]
    path = sys.argv[2] if len(sys.argv) > 2 else "direct"
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    cfg = CONFIGS[name.split("_")[1]]
    if "shape" in g:
        h, w = (int(v) for v in g["shape"])
        left, right, _ = make_pair(cfg, seed=int(g["seed"]), height=h, width=w)
    else:
        left, right, _ = make_pair(cfg, seed=int(g["seed"]))
    mc = gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block, radius=cfg.radius)
    if path == "direct":
        gpu.matcher.DIRECT_LAUNCH = True
        d, c, _ = gpu.run_pipeline(left, right, mc)
    else:
        dd, cc, _ = gpu.run_pipeline_device(torch.from_numpy(left).cuda(),
                                            torch.from_numpy(right).cuda(), mc, trace=True)
        d, c = dd.cpu().numpy().astype(np.float64), cc.cpu().numpy().astype(np.float64)
    ref_d = g["disparity"].astype(np.float64)
    n, ties, desc, unexpl, other = classify_mismatches(d, ref_d, left, right, cfg.block,
                                                       cfg.d_max, return_pixels=True, c_gpu=c)
    print(f"{name}/{path}: {n} mismatches, {ties} near ties, {desc} median descendants, "
          f"{unexpl} other")
    if not other:
        return
    _, _, _, maps = CO.run_pipeline(left, right, cfg.d_max, cfg.levels, cfg.block,
                                    radius=cfg.radius, levels_out=True)
    d_hat, c_hat = O.upsample_prior(maps[1][0], maps[1][1], left.shape)
    eng = gpu.CostEngine(left.astype(np.float64), right.astype(np.float64), cfg.block, cfg.d_max)
    gd_hat, gc_hat = gpu.upsample_prior(maps[1][0], maps[1][1], left.shape)
    tf_d, tf_c = gpu.match_level_with_prior(eng, gd_hat, gc_hat, 0.9, 0.9, cfg.radius)
    e = O.Engine(left, right, cfg.block, cfg.d_max)
    H, W = left.shape
    r = cfg.radius
    for i, j in other:
        row = e.dsi_rows(np.array([i]), np.array([j]))[0]
        ctr = int(d_hat[i, j])
        trusted = c_hat[i, j] > 0.9 and ctr + r >= 0 and ctr - r <= cfg.d_max
        if trusted:
            zs = [z for z in range(ctr - r, ctr + r + 1) if 0 <= z <= cfg.d_max]
            cand = sorted(((row[z], z) for z in zs), reverse=True)
        else:
            cand = sorted(((row[z], z) for z in range(cfg.d_max + 1)), reverse=True)
        c_sel = cand[0][0]
        nb = [(i + p, j + q) for p in (-1, 0, 1) for q in (-1, 0, 1) if 0 <= i + p < H and 0 <= j + q < W]
        s = e.dsi_rows(np.array([a for a, _ in nb]), np.array([b for _, b in nb])).sum(0) / len(nb)
        top = np.argsort(-s, kind="stable")[:2]
        print(f"  ({i},{j}) gpu d={d[i, j]:.0f} c={c[i, j]:.6f} | ref d={ref_d[i, j]:.0f} | "
              f"teacher-forced d={tf_d[i, j]:.0f} | prior d_hat={d_hat[i, j]:.0f} "
              f"c_hat-beta={c_hat[i, j] - 0.9:+.2e} gpu c_hat-beta={gc_hat[i, j] - 0.9:+.2e} "
              f"trusted={trusted} | sel top2 {cand[0][1]}:{cand[0][0]:.6f} "
              f"{cand[1][1] if len(cand) > 1 else -1}:{cand[1][0] if len(cand) > 1 else 0:.6f} "
              f"C_sel-alpha={c_sel - 0.9:+.2e} | refine top2 {top[0]}:{s[top[0]]:.6f} "
              f"{top[1]}:{s[top[1]]:.6f}")


if __name__ == "__main__":
    main()
