"""Generate golden vectors from the REAL reference package (run in the build
container only; /root/reference does not exist on the GPU box).

    python tools/make_golden.py            # writes tests/golden/*.npz

The reference ``pyrstereo`` is imported from /root/reference/pkg/src.  Its
prior window is hard-coded to +-1 (matcher.py:280,294); for the BASELINE
radii (2, 3) this script drives the reference's own stage functions
(CostEngine.at / dsi_rows, refine_level, selective_median, upsample_prior,
build_pyramid) with a radius-generalised copy of select_with_prior's control
flow, and checks at radius 1 that this driver reproduces run_pipeline
bit-for-bit.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import pyrstereo as ref  # noqa: E402
from pyrstereo import matcher as ref_matcher  # noqa: E402
from pyrstereo import pyramid as ref_pyramid  # noqa: E402
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair  # noqa: E402

COUNT_KEYS = ("trusted", "trusted_evals", "trusted_window_max",
              "full_search_pixels", "selection_evals", "refined",
              "refine_evals", "median_replaced")


def select_r(engine, d_hat, c_hat, beta, r):
    """matcher.py:263-320 with offsets range(-r, r+1)."""
    h, w = c_hat.shape
    d_max = engine.d_max
    finite = np.isfinite(d_hat)
    center = np.where(finite, d_hat, 0.0).astype(np.intp)
    window_ok = finite & (center + r >= 0) & (center - r <= d_max)
    trusted = (c_hat > beta) & window_ok
    disparity = np.empty((h, w))
    cost = np.empty((h, w))
    stats = ref_matcher.SelectionStats(trusted=int(trusted.sum()))
    before = engine.counter.count
    if stats.trusted:
        ti, tj = np.nonzero(trusted)
        tz = center[ti, tj]
        best_c = np.full(ti.shape[0], -2.0)
        best_z = np.zeros(ti.shape[0], dtype=np.intp)
        ws = np.zeros(ti.shape[0], dtype=np.intp)
        for off in range(-r, r + 1):
            z = tz + off
            legal = (z >= 0) & (z <= d_max)
            if not legal.any():
                continue
            ws[legal] += 1
            c = engine.at(ti[legal], tj[legal], z[legal])
            improve = c > best_c[legal]
            sel = np.nonzero(legal)[0][improve]
            best_c[sel] = c[improve]
            best_z[sel] = z[legal][improve]
        disparity[ti, tj] = best_z.astype(np.float64)
        cost[ti, tj] = best_c
        stats.window_max = int(ws.max())
        stats.trusted_evals = engine.counter.count - before
    full = ~trusted
    stats.full_search_pixels = int(full.sum())
    if stats.full_search_pixels:
        fi, fj = np.nonzero(full)
        rows = engine.dsi_rows(fi, fj)
        best = np.argmax(rows, axis=1)
        disparity[fi, fj] = best.astype(np.float64)
        cost[fi, fj] = rows[np.arange(fi.shape[0]), best]
    stats.evals = engine.counter.count - before
    return disparity, cost, stats


def pipeline_r(left, right, config, r):
    """run_pipeline (matcher.py:398-466) with select_r at finer levels."""
    pyr = ref.build_pyramid(left, right, config.d_max, levels=config.levels,
                            base_block=config.block)
    counter = ref.EvalCounter()
    trace = ref.PipelineTrace()

    def mk(level):
        return ref.LevelTrace(level=level.index, height=level.shape[0],
                              width=level.shape[1], d_max=level.d_max,
                              block=level.block)

    coarse = pyr.coarsest
    eng = ref.CostEngine(coarse.left, coarse.right, coarse.block, coarse.d_max,
                         sigma_eps=config.sigma_eps, sign=config.sign,
                         counter=counter)
    lt = mk(coarse)
    d, c = ref_matcher._process_level(eng, lt, config.alpha,
                                      lambda: ref.match_coarsest(eng))
    lt.full_search_pixels = lt.pixels
    lt.selection_evals = lt.pixels * (coarse.d_max + 1)
    trace.levels.append(lt)
    for k in range(len(pyr) - 2, -1, -1):
        lv = pyr[k]
        eng = ref.CostEngine(lv.left, lv.right, lv.block, lv.d_max,
                             sigma_eps=config.sigma_eps, sign=config.sign,
                             counter=counter)
        lt = mk(lv)
        d_hat, c_hat = ref.upsample_prior(d, c, lv.shape)
        box = []

        def sel():
            dd, cc, st = select_r(eng, d_hat, c_hat, config.beta, r)
            box.append(st)
            return dd, cc

        d, c = ref_matcher._process_level(eng, lt, config.alpha, sel)
        st = box[0]
        lt.trusted = st.trusted
        lt.trusted_evals = st.trusted_evals
        lt.trusted_window_max = st.window_max
        lt.full_search_pixels = st.full_search_pixels
        lt.selection_evals = st.evals
        trace.levels.append(lt)
    return d, c, trace


def counts_array(trace):
    return np.array([[lt.level, lt.height, lt.width, lt.d_max, lt.block]
                     + [getattr(lt, k) for k in COUNT_KEYS]
                     for lt in trace.levels], dtype=np.int64)


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def pipeline_case(name, left, right, d_max, levels, block, r, sign="middlebury",
                  alpha=0.9, beta=0.9):
    cfg = ref.MatchConfig(d_max=d_max, levels=levels, block=block, alpha=alpha,
                          beta=beta, sign=sign)
    t0 = time.perf_counter()
    if r == 1:
        d, c, tr = ref.run_pipeline(left, right, cfg)
        d2, c2, tr2 = pipeline_r(left, right, cfg, 1)
        assert np.array_equal(d, d2) and np.array_equal(c, c2)
        assert tr.counts_dict() == tr2.counts_dict()
    else:
        d, c, tr = pipeline_r(left, right, cfg, r)
    dt = time.perf_counter() - t0
    print(f"{name}: {left.shape} D={d_max} K={levels} b={block} r={r} "
          f"{dt:.1f}s total_evals={tr.total_evals}")
    save(f"pipe_{name}.npz", left=left, right=right, disparity=d.astype(np.int16),
         cost=c, counts=counts_array(tr),
         params=np.array([d_max, levels, block, r, 1 if sign == "paper" else 0]),
         gates=np.array([alpha, beta]), ref_seconds=np.array(dt))


def full_case(name, cfg, seed):
    """Full-size BASELINE config through the real reference (radius-generalised
    driver).  The images are not stored: the tests regenerate them with the
    seeded generator (synthetic.make_pair); only the outputs are kept (cost
    as float32, well inside the 1e-4 parity tolerance)."""
    left, right, _ = make_pair(cfg, seed=seed)
    rcfg = ref.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block)
    t0 = time.perf_counter()
    d, c, tr = pipeline_r(left, right, rcfg, cfg.radius)
    dt = time.perf_counter() - t0
    print(f"full_{name}: {left.shape} {dt:.1f}s total_evals={tr.total_evals}")
    save(f"full_{name}.npz", disparity=d.astype(np.int16), cost=c.astype(np.float32),
         counts=counts_array(tr), seed=np.array(seed),
         params=np.array([cfg.d_max, cfg.levels, cfg.block, cfg.radius, 0]),
         ref_seconds=np.array(dt))


def crop_case(name, cfg, height, width):
    """A large crop of a BASELINE config through the real reference, stored
    like full_case (outputs only; the tests regenerate the images with
    make_pair(cfg, height=, width=))."""
    left, right, _ = make_pair(cfg, height=height, width=width)
    rcfg = ref.MatchConfig(d_max=cfg.d_max, levels=cfg.levels, block=cfg.block)
    t0 = time.perf_counter()
    d, c, tr = pipeline_r(left, right, rcfg, cfg.radius)
    dt = time.perf_counter() - t0
    print(f"crop_{name}: {left.shape} {dt:.1f}s total_evals={tr.total_evals}")
    save(f"crop_{name}_{width}x{height}.npz", disparity=d.astype(np.int16),
         cost=c.astype(np.float32), counts=counts_array(tr), seed=np.array(cfg.seed),
         shape=np.array([height, width]),
         params=np.array([cfg.d_max, cfg.levels, cfg.block, cfg.radius, 0]),
         ref_seconds=np.array(dt))


def oracle_c5_case(threads=0):
    """Full-size C5 (8192x6144, D=512) through the C/OpenMP oracle, which
    reproduces every reference golden exactly (tests/test_oracle_c.py); the
    reference itself would need ~0.5 TB of host RAM here.  Stored: int16
    disparities (whole image), float32 costs on 384 stratified rows (one per
    16-row group, all 16 phases), counters."""
    from oracle import c_oracle as CO
    cfg = CONFIGS["C5"]
    left, right, _ = make_pair(cfg)
    t0 = time.perf_counter()
    d, c, counts = CO.run_pipeline(left, right, cfg.d_max, cfg.levels, cfg.block,
                                   radius=cfg.radius, threads=threads)
    dt = time.perf_counter() - t0
    h = d.shape[0]
    rows = np.arange(0, h, 16) + (np.arange(h // 16) * 7) % 16
    print(f"oracle_C5: {left.shape} {dt:.1f}s total_evals={counts[:, 9].sum() + counts[:, 11].sum()}")
    save("oracle_C5.npz", disparity=d.astype(np.int16), cost=c[rows].astype(np.float32),
         cost_rows=rows, counts=counts, seed=np.array(cfg.seed),
         params=np.array([cfg.d_max, cfg.levels, cfg.block, cfg.radius, 0]),
         oracle_seconds=np.array(dt))


def stage_cases():
    rng = np.random.default_rng(20261019)
    out = {}
    # gaussian_downsample (pyramid.py:71-81)
    for i, shp in enumerate([(8, 8), (7, 9), (31, 17), (64, 48)]):
        img = rng.random(shp) * 255.0
        out[f"down_in_{i}"] = img
        out[f"down_out_{i}"] = ref.gaussian_downsample(img)
    # CostEngine stats (zncc.py:185-189)
    for i, (shp, b) in enumerate([((12, 15), 3), ((20, 17), 5), ((16, 16), 9)]):
        img = rng.random(shp) * 255.0
        e = ref.CostEngine(img, img, b, 4)
        out[f"stats_in_{i}"] = img
        out[f"stats_b_{i}"] = np.array(b)
        out[f"stats_mean_{i}"] = e.mean_l
        out[f"stats_sigma_{i}"] = e.sigma_l
    # upsample_prior incl. the scipy cubic B-spline (matcher.py:236-260)
    for i, (ch, cw, h, w) in enumerate([(4, 5, 8, 10), (5, 6, 9, 11),
                                        (47, 57, 94, 113), (94, 113, 188, 225)]):
        dc = rng.integers(0, 40, size=(ch, cw)).astype(np.float64)
        cc = np.clip(rng.normal(0.7, 0.4, size=(ch, cw)), -1, 1)
        dh, chat = ref.upsample_prior(dc, cc, (h, w))
        out[f"up_d_{i}"] = dc
        out[f"up_c_{i}"] = cc
        out[f"up_shape_{i}"] = np.array([h, w])
        out[f"up_dhat_{i}"] = dh
        out[f"up_chat_{i}"] = chat
    # selective_median (criterion-7 style, matcher.py:323-359)
    med_d, med_c, med_a, med_out = [], [], [], []
    mrng = np.random.default_rng(1007)
    for _ in range(100):
        dd = mrng.integers(0, 20, size=(9, 9)).astype(float)
        cc = mrng.uniform(-1.0, 1.0, size=(9, 9))
        a = float(mrng.uniform(0.2, 0.95))
        med_d.append(dd), med_c.append(cc), med_a.append(a)
        med_out.append(ref.selective_median(dd, cc, a))
    out["med_d"] = np.array(med_d)
    out["med_c"] = np.array(med_c)
    out["med_alpha"] = np.array(med_a)
    out["med_out"] = np.array(med_out)
    # coarse full search (criterion-1 style, matcher.py:184-193)
    frng = np.random.default_rng(1001)
    for i in range(24):
        h = int(frng.integers(16, 33))
        w = int(frng.integers(16, 33))
        d_max = int(frng.integers(4, 11))
        block = int(frng.choice([3, 5]))
        left, right = frng.random((h, w)), frng.random((h, w))
        sign = "paper" if i % 4 == 3 else "middlebury"
        e = ref.CostEngine(left, right, block=block, d_max=d_max, sign=sign)
        d, c = ref.match_coarsest(e)
        out[f"full_l_{i}"] = left
        out[f"full_r_{i}"] = right
        out[f"full_p_{i}"] = np.array([d_max, block, 1 if sign == "paper" else 0])
        out[f"full_d_{i}"] = d
        out[f"full_c_{i}"] = c
    # select_with_prior r=1 and refine_level on a shifted pair
    srng = np.random.default_rng(7)
    left, right = ref.shifted_pair(24, 40, 5, srng, cutoff=0.1)
    e = ref.CostEngine(left, right, block=5, d_max=12)
    d_hat = np.clip(np.round(5 + srng.normal(0, 2, size=(24, 40))), -3, 15)
    d_hat[3, 4] = np.nan
    c_hat = srng.uniform(0.5, 1.0, size=(24, 40))
    d, c, st = ref.select_with_prior(e, d_hat, c_hat, 0.9)
    out.update(sel_l=left, sel_r=right, sel_dhat=d_hat, sel_chat=c_hat,
               sel_d=d, sel_c=c,
               sel_stats=np.array([st.trusted, st.trusted_evals, st.window_max,
                                   st.full_search_pixels, st.evals]))
    e2 = ref.CostEngine(left, right, block=5, d_max=12)
    rd, rc = ref.refine_level(e2, d, c, 0.9)
    out.update(ref_d=rd, ref_c=rc, ref_evals=np.array(e2.counter.count))
    save("stages.npz", **out)


def stage_api_cases():
    """Stage APIs off run_pipeline's path:
    CostEngine.plane / full_volume (zncc.py:202-249), dsi_entry,
    dsi_slice, averaged_dsi (zncc.py:304-350), the EvalCounter tally of each
    call, match_level_with_prior (matcher.py:362-369) and binomial_smooth
    (pyramid.py:65-68)."""
    out = {}
    rng = np.random.default_rng(20261020)
    # plane / full_volume on random textures (both sign conventions), incl.
    # a flat (degenerate) patch so the -1 floor of sigma < eps is pinned
    for i, (h, w, b, d, sign) in enumerate([(8, 10, 3, 5, "middlebury"),
                                            (16, 16, 5, 8, "middlebury"),
                                            (13, 21, 3, 7, "paper"),
                                            (24, 31, 7, 12, "middlebury")]):
        left, right = rng.random((h, w)), rng.random((h, w))
        left[2:6, 2:6] = 0.5
        e = ref.CostEngine(left, right, block=b, d_max=d, sign=sign)
        vol = e.full_volume()
        out[f"vol_l_{i}"], out[f"vol_r_{i}"] = left, right
        out[f"vol_p_{i}"] = np.array([b, d, 1 if sign == "paper" else 0])
        out[f"vol_{i}"] = vol
        out[f"vol_count_{i}"] = np.array(e.counter.count)
    # dsi_entry / dsi_slice / averaged_dsi on a shifted pair
    left, right = ref.shifted_pair(9, 12, 2, rng, cutoff=0.2)
    e = ref.CostEngine(left, right, block=3, d_max=4)
    pts = [(4, 6, 2), (0, 0, 0), (8, 11, 4), (3, 1, 3), (5, 9, 1)]
    out["pt_l"], out["pt_r"] = left, right
    out["pt_ijz"] = np.array(pts)
    out["pt_entry"] = np.array([ref.dsi_entry(e, i, j, z) for i, j, z in pts])
    out["pt_slice"] = np.array([e.dsi_slice(i, j).costs for i, j, _ in pts])
    far = [(-5, -5), (-6, 0), (0, -9)]
    out["pt_avg"] = np.array([ref.averaged_dsi(e, i, j).costs for i, j, _ in pts])
    out["pt_avg_far"] = ref.averaged_dsi(e, 0, 0, neighborhood=far).costs
    out["pt_count"] = np.array(e.counter.count)
    # match_level_with_prior (r = 1, the reference's own) on a shifted pair
    srng = np.random.default_rng(8)
    left, right = ref.shifted_pair(32, 48, 6, srng, cutoff=0.1)
    e = ref.CostEngine(left, right, block=5, d_max=14)
    d_hat = np.clip(np.round(6 + srng.normal(0, 2, size=(32, 48))), -3, 17)
    d_hat[5, 7] = np.nan
    c_hat = srng.uniform(0.6, 1.0, size=(32, 48))
    md, mc = ref.match_level_with_prior(e, d_hat, c_hat, 0.9, 0.9)
    out.update(ml_l=left, ml_r=right, ml_dhat=d_hat, ml_chat=c_hat, ml_d=md, ml_c=mc,
               ml_count=np.array(e.counter.count))
    # binomial_smooth (full resolution, no decimation)
    for i, shp in enumerate([(5, 7), (2, 2), (33, 18)]):
        img = rng.random(shp) * 255.0
        out[f"bs_in_{i}"] = img
        out[f"bs_out_{i}"] = ref_pyramid.binomial_smooth(img)
    save("stage_api.npz", **out)


def scoring_cases():
    """baseline.py / evaluation.py / synthetic.py vectors."""
    out = {}
    rng = np.random.default_rng(31)
    left, right = ref.shifted_pair(24, 40, 4, rng, cutoff=0.15)
    out.update(sp_left=left, sp_right=right,
               sp_mask=ref.interior_mask(left.shape, 4, 5),
               sp_mask_x=ref.interior_mask((30, 41), 3, 11, extra=2))
    d, c, n = ref.baseline_bm(left, right, 8, 5)
    out.update(bm_d=d, bm_c=c, bm_evals=np.array(n))
    rng = np.random.default_rng(32)
    l2 = rng.random((18, 26))
    r2 = np.roll(l2, -3, axis=1) + 0.01 * rng.random((18, 26))
    l2[4:10, 6:14] = 0.5                       # flat blocks -> degenerate ZNCC
    d, c, n = ref.baseline_bm(l2, r2, 6, 3, sign="middlebury")
    out.update(bm2_left=l2, bm2_right=r2, bm2_d=d, bm2_c=c, bm2_evals=np.array(n))
    d, c, n = ref.baseline_bm(r2, l2, 6, 7, sign="paper")
    out.update(bm3_d=d, bm3_c=c, bm3_evals=np.array(n))
    d, c, n = ref.baseline_bm(l2, r2, 0, 3)
    out.update(bm4_d=d, bm4_c=c, bm4_evals=np.array(n))
    # evaluate: random maps with NaN outputs and invalid reference pixels
    rng = np.random.default_rng(33)
    ev_d = rng.uniform(0, 40, (37, 53))
    ev_d[rng.random(ev_d.shape) < 0.07] = np.nan
    ev_d[0, :5] = np.inf
    ev_g = ev_d + rng.normal(0, 3, ev_d.shape)
    ev_inv = rng.random(ev_d.shape) < 0.1
    ev_g[ev_inv] = np.nan
    gt = ref.GroundTruthDisparity(values=ev_g, invalid=ev_inv)
    rows = []
    for scale in (1.0, 0.5, 2.0):
        r = ref.evaluate(ev_d, gt, scale=scale)
        rows.append([scale, r.bad_1, r.bad_2, r.bad_4, r.avg_abs_err, r.evaluated,
                     r.gt_invalid, r.output_invalid])
    out.update(ev_d=ev_d, ev_g=ev_g, ev_inv=ev_inv, ev_reports=np.array(rows))
    save("scoring.npz", **out)


def formats_cases():
    """formats.py codecs: files written by the reference writers and
    hand-built PNM variants, with the reference readers' decoded arrays;
    malformed inputs with the reference's exception class."""
    import tempfile
    from pyrstereo import formats as F
    out = {}
    tmp = tempfile.mkdtemp()
    rng = np.random.default_rng(41)
    files = {}
    v = rng.random((9, 13))
    v[2, 3] = np.nan
    for name, kw in [("pfm_le", dict(scale=-1.0)), ("pfm_be", dict(scale=1.0)),
                     ("pfm_s2", dict(scale=-2.5))]:
        F.write_pfm(v, os.path.join(tmp, name), **kw)
    dsp = rng.uniform(0, 70, (11, 6))
    dsp[0, 0] = np.nan
    dsp[1, 1] = np.inf
    dsp[2, 2] = -5.0
    dsp[3, 3] = 1e9
    F.write_pgm(v, os.path.join(tmp, "pgm8"))
    F.write_pgm(dsp, os.path.join(tmp, "pgm_preview"), scale_max=70.0)
    F.write_pgm(v, os.path.join(tmp, "pgm16"), maxval=4095)
    F.write_pgm(np.array([[0.5 / 255, 1.5 / 255, 2.5 / 255, 253.5 / 255]]),
                os.path.join(tmp, "pgm_half"))
    for name in ("pfm_le", "pfm_be", "pfm_s2", "pgm8", "pgm_preview", "pgm16", "pgm_half"):
        files[name] = open(os.path.join(tmp, name), "rb").read()
    img = rng.integers(0, 256, (7, 10))
    rgb = rng.integers(0, 1024, (5, 6, 3))
    files["p5"] = b"P5\n# comment\n10 7\n255\n" + img.astype("u1").tobytes()
    files["p2"] = (b"P2\n10 7 255\n" + " ".join(str(x) for x in img.ravel()).encode() + b"\n")
    files["p6_16"] = b"P6 6 5\n1023\n" + rgb.astype(">u2").tobytes()
    files["p3"] = (b"P3\n6 5\n# c\n1023\n" + " ".join(str(x) for x in rgb.ravel()).encode())
    files["p6_8"] = b"P6\n6 5\n255\n" + (rgb % 256).astype("u1").tobytes()
    for name, data in files.items():
        out[f"file_{name}"] = np.frombuffer(data, dtype=np.uint8)
        path = os.path.join(tmp, name)
        open(path, "wb").write(data)
        if name.startswith("pfm"):
            g = F.read_pfm(path)
            out[f"dec_{name}"] = g.values
            out[f"inv_{name}"] = g.invalid
        else:
            out[f"dec_{name}"] = F.read_pnm(path)
    out["src_v"] = v
    out["src_dsp"] = dsp
    bad = [b"P7\n2 2\n255\n" + bytes(4), b"P5\n2 x\n255\n" + bytes(4),
           b"P5\n2 2\n255\n" + bytes(3), b"P2\n2 2\n255\n1 2 3\n",
           b"P5\n2 2\n0\n" + bytes(4), b"P5\n2 2\n70000\n" + bytes(16), b"P5\n2 2\n255",
           b"P2\n2 2\n100\n1 2 3 101\n", b"P5\n2 2\n100\n" + bytes([0, 50, 100, 255]),
           b"P5\n0 2\n255\n" + bytes(4), b"P2\n2 2\n9\n1 x 3 4\n", b"P5 2 2 255" + bytes(4),
           b"", b"# only a comment\n",
           b"PF\n1 1\n-1.0\n" + bytes(12), b"Pf\n1 1\n0.0\n" + bytes(4),
           b"Pf\n2 2\n-1.0\n" + bytes(8), b"Pf\n2 2\nabc\n" + bytes(16),
           b"Pf\n-2 2\n-1.0\n" + bytes(16), b"Pf\n1 1\n-1.0" + bytes(4)]
    kinds, msgs = [], []
    for k, data in enumerate(bad):
        path = os.path.join(tmp, f"bad{k}")
        open(path, "wb").write(data)
        reader = F.read_pfm if data.startswith(b"P") and data[1:2] in (b"f", b"F") else F.read_pnm
        try:
            reader(path)
            kinds.append("none")
            msgs.append("")
        except Exception as e:   # noqa: BLE001
            kinds.append(type(e).__name__)
            msgs.append(str(e))
        out[f"bad_{k}"] = np.frombuffer(data, dtype=np.uint8)
    out["bad_kind"] = np.array(kinds)
    out["bad_msg"] = np.array(msgs)
    save("formats.npz", **out)


def main():
    os.makedirs(OUT, exist_ok=True)
    if sys.argv[1:] == ["scoring"]:
        scoring_cases()
        return
    if sys.argv[1:] == ["formats"]:
        formats_cases()
        return
    if sys.argv[1:] == ["stage_api"]:
        stage_api_cases()
        return
    if sys.argv[1:] == ["full"]:   # full-size C2 and one C4 pair (minutes)
        full_case("C2", CONFIGS["C2"], CONFIGS["C2"].seed)
        full_case("C4", CONFIGS["C4"], CONFIGS["C4"].seed)
        return
    if sys.argv[1:] == ["oracle_C5"]:   # full C5 via the C oracle (about 80 s on 8 cores)
        oracle_c5_case()
        return
    if sys.argv[1:] == ["crop_C5"]:   # 2048x1536 C5 crop (about 16 min, 35 GB)
        crop_case("C5", CONFIGS["C5"], 1536, 2048)
        return
    if sys.argv[1:] == ["full_C3"]:   # full-size C3 (about 9 min, 8 GB)
        full_case("C3", CONFIGS["C3"], CONFIGS["C3"].seed)
        return
    scoring_cases()
    formats_cases()
    stage_cases()
    rng = np.random.default_rng(16)
    left, right = ref.shifted_pair(64, 64, 6, rng, cutoff=0.05)
    pipeline_case("shift64_b11", left, right, 16, 2, 11, 1)
    rng = np.random.default_rng(20)
    r_, l_ = ref.shifted_pair(64, 64, 5, rng, cutoff=0.05)
    pipeline_case("paper64_b11", l_, r_, 16, 2, 11, 1, sign="paper")
    rng = np.random.default_rng(19)
    left, right = ref.shifted_pair(48, 56, 4, rng, cutoff=0.05)
    pipeline_case("shift48_k0", left, right, 12, 0, 5, 1)
    # BASELINE C1 at full size: r=1 (reference run_pipeline) and r=2
    l1, r1, _ = make_pair(CONFIGS["C1"])
    pipeline_case("C1_r1", l1, r1, 64, 2, 5, 1)
    pipeline_case("C1_r2", l1, r1, 64, 2, 5, 2)
    # parity-size crops of the other configs at their own parameters
    crops = {"C2": (248, 368), "C3": (248, 368), "C4": (180, 320),
             "C5": (384, 512)}
    for name, (h, w) in crops.items():
        cfg = CONFIGS[name]
        lc, rc, _ = make_pair(cfg, height=h, width=w)
        pipeline_case(f"{name}crop", lc, rc, cfg.d_max, cfg.levels, cfg.block,
                      cfg.radius)


if __name__ == "__main__":
    main()
