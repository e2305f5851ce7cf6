"""CPU oracle for the MSHBM disparity hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy float64, the algorithm of the reference
package ``pyrstereo`` (``/root/reference/pkg/src/pyrstereo``) along the path
``run_pipeline`` walks.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product path (``paper_1901_09593_b200``) never calls into it.

Differences from the reference, all deliberate:

* ``radius`` generalises the hard-coded +-1 prior window of
  ``select_with_prior`` (``matcher.py:280,294``); at radius=1 the restatement
  is the reference algorithm (pinned by ``tests/golden``).
* third-party numerics are restated instead of imported:
  ``scipy.ndimage.correlate1d`` (binomial smoothing), ``uniform_filter``
  (box means), ``binary_dilation`` (3x3), ``map_coordinates(order=3,
  mode='nearest')`` (cubic B-spline with 12-sample edge pre-padding, scipy
  1.18.1 ``_prepad_for_spline_filter`` + ``spline_filter1d`` with the
  'nearest'/'reflect' causal/anticausal initialisation).  These agree with
  scipy to ~1e-13 (checked in tests/test_oracle_golden.py).
* full-range DSI rows are reduced per chunk / per row band (argmax, 3x3
  sums) instead of being materialised whole (``zncc.py:295``), so large
  configs fit in host memory.  Per-pixel arithmetic is the reference's
  ``CostEngine._gather`` (``zncc.py:271-287``) unchanged.
* ``workers`` threads evaluate independent chunks; results do not depend on
  the worker count (the chunk composition is fixed).

Parity status: pinned against the reference itself (golden vectors made by
``tools/make_golden.py`` importing /root/reference) -- see DESIGN.md.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

MIDDLEBURY = "middlebury"
PAPER = "paper"
_CHUNK = 32768                      # zncc.py:52 _GATHER_CHUNK
_BINOMIAL = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 16.0   # pyramid.py:30


# --------------------------------------------------------------------------
# pyramid (pyramid.py:65-160)
# --------------------------------------------------------------------------

def correlate1d_nearest(img: np.ndarray, weights: np.ndarray, axis: int) -> np.ndarray:
    """scipy.ndimage.correlate1d(img, w, axis, mode='nearest') restated."""
    r = weights.shape[0] // 2
    pad = [(0, 0)] * img.ndim
    pad[axis] = (r, r)
    p = np.pad(img, pad, mode="edge")
    n = img.shape[axis]
    out = np.zeros(img.shape, dtype=np.float64)
    for t in range(weights.shape[0]):
        sl = [slice(None)] * img.ndim
        sl[axis] = slice(t, t + n)
        out += weights[t] * p[tuple(sl)]
    return out


def binomial_smooth(img):
    """pyramid.py:65-68: axis 0 then axis 1, replicate borders."""
    out = correlate1d_nearest(np.asarray(img, np.float64), _BINOMIAL, 0)
    return correlate1d_nearest(out, _BINOMIAL, 1)


def gaussian_downsample(img):
    """pyramid.py:71-81: smooth, keep even rows/cols (ceil halving)."""
    img = np.asarray(img, dtype=np.float64)
    if img.ndim != 2 or img.shape[0] < 2 or img.shape[1] < 2:
        raise ValueError(f"cannot downsample image of shape {img.shape}")
    return binomial_smooth(img)[::2, ::2]


def level_d_max(d_max, k):          # pyramid.py:84-86
    return max(1, d_max >> k)


def level_block(base_block, k):     # pyramid.py:89-94
    b = base_block >> k
    if b % 2 == 0:
        b -= 1
    return max(b, 3)


def auto_levels(width, height, d_max, base_block):   # pyramid.py:97-112
    if min(width, height) <= 0 or d_max < 1 or base_block < 1:
        raise ValueError("width, height, d_max and base_block must be positive")
    k = 0
    while (min(width, height) / 2 ** (k + 1) >= 4 * base_block
           and d_max >> (k + 1) >= 2):
        k += 1
    return k


def build_pyramid(left, right, d_max, levels=None, base_block=11):
    """pyramid.py:115-160. Returns list of (left, right, d_max, block)."""
    left = np.asarray(left, dtype=np.float64)
    right = np.asarray(right, dtype=np.float64)
    if left.ndim != 2 or left.shape != right.shape:
        raise ValueError(f"left/right shapes differ: {left.shape} vs {right.shape}")
    height, width = left.shape
    if levels is None:
        levels = auto_levels(width, height, d_max, base_block)
    if levels > 0:
        h, w = height, width
        for _ in range(levels):
            h, w = (h + 1) // 2, (w + 1) // 2
        if min(h, w) < 2 * level_block(base_block, levels):
            raise ValueError("pyramid too deep for the image")
        if d_max >> levels < 2:
            raise ValueError("pyramid too deep for the disparity range")
    out = [(left, right, level_d_max(d_max, 0), level_block(base_block, 0))]
    cl, cr = left, right
    for k in range(1, levels + 1):
        cl, cr = gaussian_downsample(cl), gaussian_downsample(cr)
        out.append((cl, cr, level_d_max(d_max, k), level_block(base_block, k)))
    return out


# --------------------------------------------------------------------------
# cost engine (zncc.py:144-319)
# --------------------------------------------------------------------------

def box_mean_nearest(img, size):
    """scipy uniform_filter(img, size, mode='nearest') restated (per axis)."""
    w = np.full(size, 1.0 / size)
    out = correlate1d_nearest(img, w, 0)
    return correlate1d_nearest(out, w, 1)


class Engine:
    """Restatement of ``CostEngine`` (zncc.py:144-307) for one level."""

    def __init__(self, left, right, block, d_max, sigma_eps=1e-6,
                 sign=MIDDLEBURY, workers=1):
        left = np.ascontiguousarray(left, dtype=np.float64)
        right = np.ascontiguousarray(right, dtype=np.float64)
        self.height, self.width = left.shape
        self.block, self.half, self.area = block, block // 2, block * block
        self.d_max = int(d_max)
        self.sigma_eps = float(sigma_eps)
        self.sign = sign
        self.workers = max(1, int(workers))
        self.count = 0
        self._lp = np.pad(left, self.half, mode="edge")
        self._rp = np.pad(right, self.half, mode="edge")
        self._lwin = sliding_window_view(self._lp, (block, block))
        self._rwin = sliding_window_view(self._rp, (block, block))
        self.mean_l, self.sigma_l = self._stats(left)
        self.mean_r, self.sigma_r = self._stats(right)
        self._ok_l = self.sigma_l >= self.sigma_eps
        self._ok_r = self.sigma_r >= self.sigma_eps

    def _stats(self, img):                              # zncc.py:185-189
        mean = box_mean_nearest(img, self.block)
        mean_sq = box_mean_nearest(img * img, self.block)
        return mean, np.sqrt(np.maximum(mean_sq - mean * mean, 0.0))

    def _right_cols(self, j, z):                        # zncc.py:191-194
        return j - z if self.sign == MIDDLEBURY else j + z

    def plane(self, z):
        """zncc.py:202-231: one disparity plane via integral-image box sums."""
        h, w, b = self.height, self.width, self.block
        lp, rp = self._lp, self._rp
        prod = np.zeros_like(lp)
        if z == 0:
            np.multiply(lp, rp, out=prod)
        elif self.sign == MIDDLEBURY:
            np.multiply(lp[:, z:], rp[:, :-z], out=prod[:, z:])
        else:
            np.multiply(lp[:, :-z], rp[:, z:], out=prod[:, :-z])
        integral = np.zeros((prod.shape[0] + 1, prod.shape[1] + 1))
        integral[1:, 1:] = prod.cumsum(axis=0).cumsum(axis=1)
        cross = (integral[b:, b:] - integral[:-b, b:]
                 - integral[b:, :-b] + integral[:-b, :-b])
        cols = self._right_cols(np.arange(w), z)
        in_range = (cols >= 0) & (cols <= w - 1)
        safe = np.clip(cols, 0, w - 1)
        mean_r = self.mean_r[:, safe]
        sigma_r = self.sigma_r[:, safe]
        ok = self._ok_l & self._ok_r[:, safe] & in_range[np.newaxis, :]
        cov = cross / self.area - self.mean_l * mean_r
        denom = np.where(ok, self.sigma_l * sigma_r, 1.0)
        self.count += h * w
        return np.where(ok, np.clip(cov / denom, -1.0, 1.0), -1.0)

    def gather(self, rows, cols, z):
        """zncc.py:271-287: direct block products for (row, col, z) triples."""
        w = self.width
        rcols = self._right_cols(cols, z)
        in_range = (rcols >= 0) & (rcols <= w - 1)
        safe = np.clip(rcols, 0, w - 1)
        lpat = self._lwin[rows, cols]
        rpat = self._rwin[rows, safe]
        cross = np.einsum("spq,spq->s", lpat, rpat)
        mean_r = self.mean_r[rows, safe]
        sigma_r = self.sigma_r[rows, safe]
        ok = self._ok_l[rows, cols] & self._ok_r[rows, safe] & in_range
        cov = cross / self.area - self.mean_l[rows, cols] * mean_r
        denom = np.where(ok, self.sigma_l[rows, cols] * sigma_r, 1.0)
        return np.where(ok, np.clip(cov / denom, -1.0, 1.0), -1.0)

    def at(self, rows, cols, z):
        """zncc.py:251-269 (counts every triple)."""
        rows = np.asarray(rows, np.intp).ravel()
        cols = np.asarray(cols, np.intp).ravel()
        z = np.asarray(z, np.intp).ravel()
        out = np.empty(rows.shape[0])
        for s in range(0, rows.shape[0], _CHUNK):
            sl = slice(s, s + _CHUNK)
            out[sl] = self.gather(rows[sl], cols[sl], z[sl])
        self.count += rows.shape[0]
        return out

    def _dsi_chunk(self, r, c):
        out = np.empty((r.shape[0], self.d_max + 1))
        for z in range(self.d_max + 1):
            out[:, z] = self.gather(r, c, np.full(r.shape, z, dtype=np.intp))
        return out

    def dsi_map(self, rows, cols, reduce):
        """zncc.py:289-302 with a per-chunk reduction instead of storing rows.

        Returns the list of ``reduce(chunk_rows)`` results in chunk order.
        """
        rows = np.asarray(rows, np.intp).ravel()
        cols = np.asarray(cols, np.intp).ravel()
        starts = list(range(0, rows.shape[0], _CHUNK))

        def job(s):
            return reduce(self._dsi_chunk(rows[s:s + _CHUNK], cols[s:s + _CHUNK]))

        if self.workers > 1 and len(starts) > 1:
            with ThreadPoolExecutor(self.workers) as pool:
                res = list(pool.map(job, starts))
        else:
            res = [job(s) for s in starts]
        self.count += rows.shape[0] * (self.d_max + 1)
        return res

    def dsi_rows(self, rows, cols):
        res = self.dsi_map(rows, cols, lambda x: x)
        if not res:
            return np.empty((0, self.d_max + 1))
        return np.concatenate(res, axis=0)


def _argmax_reduce(rows):
    best = np.argmax(rows, axis=1)
    return best, rows[np.arange(rows.shape[0]), best]


# --------------------------------------------------------------------------
# matcher stages (matcher.py:184-359)
# --------------------------------------------------------------------------

def match_coarsest(engine):
    """matcher.py:184-193: full volume, first argmax."""
    vol = np.empty((engine.d_max + 1, engine.height, engine.width))
    planes = range(engine.d_max + 1)
    if engine.workers > 1:
        with ThreadPoolExecutor(engine.workers) as pool:
            for z, p in enumerate(pool.map(engine.plane, planes)):
                vol[z] = p
    else:
        for z in planes:
            vol[z] = engine.plane(z)
    d = np.argmax(vol, axis=0)
    c = np.take_along_axis(vol, d[np.newaxis], axis=0)[0]
    return d.astype(np.float64), c


def select_with_prior(engine, d_hat, c_hat, beta, radius=1):
    """matcher.py:263-320 with the +-1 window generalised to +-radius."""
    h, w = c_hat.shape
    d_max = engine.d_max
    finite = np.isfinite(d_hat)
    center = np.where(finite, d_hat, 0.0).astype(np.intp)
    window_ok = finite & (center + radius >= 0) & (center - radius <= d_max)
    trusted = (c_hat > beta) & window_ok
    disparity = np.empty((h, w))
    cost = np.empty((h, w))
    stats = {"trusted": int(trusted.sum()), "trusted_evals": 0,
             "window_max": 0, "full_search_pixels": 0, "evals": 0}
    before = engine.count
    if stats["trusted"]:
        ti, tj = np.nonzero(trusted)
        tz = center[ti, tj]
        best_c = np.full(ti.shape[0], -2.0)
        best_z = np.zeros(ti.shape[0], dtype=np.intp)
        wsize = np.zeros(ti.shape[0], dtype=np.intp)
        for off in range(-radius, radius + 1):
            z = tz + off
            legal = (z >= 0) & (z <= d_max)
            if not legal.any():
                continue
            wsize[legal] += 1
            c = engine.at(ti[legal], tj[legal], z[legal])
            improve = c > best_c[legal]
            sel = np.nonzero(legal)[0][improve]
            best_c[sel] = c[improve]
            best_z[sel] = z[legal][improve]
        disparity[ti, tj] = best_z.astype(np.float64)
        cost[ti, tj] = best_c
        stats["window_max"] = int(wsize.max())
        stats["trusted_evals"] = engine.count - before
    full = ~trusted
    stats["full_search_pixels"] = int(full.sum())
    if stats["full_search_pixels"]:
        fi, fj = np.nonzero(full)
        res = engine.dsi_map(fi, fj, _argmax_reduce)
        best = np.concatenate([r[0] for r in res])
        bc = np.concatenate([r[1] for r in res])
        disparity[fi, fj] = best.astype(np.float64)
        cost[fi, fj] = bc
    stats["evals"] = engine.count - before
    return disparity, cost, stats


def dilate3x3(mask):
    """scipy binary_dilation(mask, ones((3,3))) with a False border."""
    h, w = mask.shape
    p = np.zeros((h + 2, w + 2), dtype=bool)
    p[1:-1, 1:-1] = mask
    out = np.zeros((h, w), dtype=bool)
    for di in range(3):
        for dj in range(3):
            out |= p[di:di + h, dj:dj + w]
    return out


def refine_level(engine, disparity, cost, alpha, band_bytes=1 << 28):
    """matcher.py:196-233, processed in row bands to bound memory."""
    low = cost <= alpha
    if not low.any():
        return disparity.copy(), cost.copy()
    h, w = cost.shape
    needed = dilate3x3(low)
    new_d = disparity.copy()
    new_c = cost.copy()
    row_bytes = max(1, w * (engine.d_max + 1) * 8)
    band = max(1, int(band_bytes // row_bytes) - 2)
    count_before = engine.count
    for r0 in range(0, h, band):
        r1 = min(h, r0 + band)
        if not low[r0:r1].any():
            continue
        q0, q1 = max(0, r0 - 1), min(h, r1 + 1)
        nmask = np.zeros_like(needed)
        nmask[q0:q1] = needed[q0:q1]
        nrows, ncols = np.nonzero(nmask)
        rows_dsi = engine.dsi_rows(nrows, ncols)
        index = np.full((h, w), -1, dtype=np.intp)
        index[nrows, ncols] = np.arange(nrows.shape[0])
        li, lj = np.nonzero(low[r0:r1])
        li = li + r0
        summed = np.zeros((li.shape[0], engine.d_max + 1))
        members = np.zeros(li.shape[0])
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                qi, qj = li + di, lj + dj
                inside = (qi >= 0) & (qi < h) & (qj >= 0) & (qj < w)
                summed[inside] += rows_dsi[index[qi[inside], qj[inside]]]
                members[inside] += 1.0
        best = np.argmax(summed, axis=1)
        new_d[li, lj] = best.astype(np.float64)
        new_c[li, lj] = summed[np.arange(li.shape[0]), best] / members
    # banding re-evaluates halo rows; the trace counts |needed| * (d+1) once,
    # exactly as the reference's single dsi_rows call does.
    engine.count = count_before + int(needed.sum()) * (engine.d_max + 1)
    return new_d, new_c


def selective_median(disparity, cost, alpha):
    """matcher.py:323-359: lower median of confident 5x5 neighbours."""
    low = cost <= alpha
    if not low.any():
        return disparity.copy()
    cpad = np.pad(cost, 2, mode="constant", constant_values=-2.0)
    dpad = np.pad(disparity, 2, mode="constant", constant_values=0.0)
    cwin = sliding_window_view(cpad, (5, 5))
    dwin = sliding_window_view(dpad, (5, 5))
    li, lj = np.nonzero(low)
    cw = cwin[li, lj].reshape(li.shape[0], 25)
    dw = dwin[li, lj].reshape(li.shape[0], 25)
    q = (cw > alpha) & np.isfinite(dw)
    counts = q.sum(axis=1)
    pool = np.where(q, dw, np.inf)
    pool.sort(axis=1)
    pick = np.maximum(counts - 1, 0) // 2
    med = pool[np.arange(li.shape[0]), pick]
    out = disparity.copy()
    have = counts > 0
    out[li[have], lj[have]] = med[have]
    return out


# --------------------------------------------------------------------------
# cubic B-spline upsampling (matcher.py:236-260 via scipy map_coordinates)
# --------------------------------------------------------------------------

_POLE = math.sqrt(3.0) - 2.0
_NPAD = 12


def _spline_filter_axis(c, axis):
    """scipy spline_filter1d(order=3, mode='nearest') along ``axis``.

    gain (1-z)(1-1/z); causal 'reflect' init, causal recursion;
    anticausal init c[n-1] *= z/(z-1); anticausal recursion.
    """
    z = _POLE
    c = np.moveaxis(c, axis, -1).copy()
    n = c.shape[-1]
    c *= (1.0 - z) * (1.0 - 1.0 / z)
    if n > 1:
        zn = z ** n
        c0 = c[..., 0].copy()
        acc = c[..., 0] + zn * c[..., n - 1]
        zi = z
        for i in range(1, n):
            acc = acc + zi * (c[..., i] + zn * c[..., n - 1 - i])
            zi *= z
            if zi == 0.0:
                break
        c[..., 0] = acc * (z / (1.0 - zn * zn)) + c0
        for i in range(1, n):
            c[..., i] += z * c[..., i - 1]
        c[..., n - 1] *= z / (z - 1.0)
        for i in range(n - 2, -1, -1):
            c[..., i] = z * (c[..., i + 1] - c[..., i])
    return np.moveaxis(c, -1, axis)


def bspline_coefficients(cost):
    """Edge pre-pad by 12, then prefilter axis 0 and axis 1 (scipy order)."""
    p = np.pad(np.asarray(cost, np.float64), _NPAD, mode="edge")
    p = _spline_filter_axis(p, 0)
    return _spline_filter_axis(p, 1)


def _bspline_weights(t):
    w0 = (1.0 - t) ** 3 / 6.0
    w1 = (4.0 - 6.0 * t * t + 3.0 * t ** 3) / 6.0
    w2 = (1.0 + 3.0 * t + 3.0 * t * t - 3.0 * t ** 3) / 6.0
    w3 = t ** 3 / 6.0
    return (w0, w1, w2, w3)


def bspline_sample(coef, y, x):
    """Cubic B-spline value at padded-array coordinates (y, x) (broadcast)."""
    fy = np.floor(y)
    fx = np.floor(x)
    wy = _bspline_weights(y - fy)
    wx = _bspline_weights(x - fx)
    iy = fy.astype(np.intp) - 1
    ix = fx.astype(np.intp) - 1
    hh, ww = coef.shape
    out = 0.0
    for a in range(4):
        ry = np.clip(iy + a, 0, hh - 1)
        row = 0.0
        for b in range(4):
            rx = np.clip(ix + b, 0, ww - 1)
            row = row + wx[b] * coef[ry, rx]
        out = out + wy[a] * row
    return out


def upsample_prior(d_coarse, c_coarse, target_shape):
    """matcher.py:236-260: 2x NN disparity, B-spline cost, clamp [-1, 1]."""
    h, w = target_shape
    ch, cw = d_coarse.shape
    if c_coarse.shape != (ch, cw):
        raise ValueError("disparity and cost maps differ in shape")
    if ch != (h + 1) // 2 or cw != (w + 1) // 2:
        raise ValueError("not the dyadic parent")
    d_hat = 2.0 * np.repeat(np.repeat(d_coarse, 2, axis=0), 2, axis=1)[:h, :w]
    yi = (np.arange(h) + 0.5) * (ch / h) - 0.5 + _NPAD
    xi = (np.arange(w) + 0.5) * (cw / w) - 0.5 + _NPAD
    coef = bspline_coefficients(c_coarse)
    c_hat = bspline_sample(coef, yi[:, None], xi[None, :])
    return d_hat, np.clip(c_hat, -1.0, 1.0)


# --------------------------------------------------------------------------
# pipeline (matcher.py:372-466)
# --------------------------------------------------------------------------

_COUNT_KEYS = ("level", "height", "width", "d_max", "block", "pixels",
               "trusted", "trusted_evals", "trusted_window_max",
               "full_search_pixels", "selection_evals", "refined",
               "refine_evals", "median_replaced")


def _process_level(engine, tr, alpha, select):
    d, c = select()
    before = engine.count
    tr["refined"] = int(np.sum(c <= alpha))
    d, c = refine_level(engine, d, c, alpha)
    tr["refine_evals"] = engine.count - before
    f = selective_median(d, c, alpha)
    both_nan = np.isnan(d) & np.isnan(f)
    tr["median_replaced"] = int(np.sum(~both_nan & (d != f)))
    return f, c


def run_pipeline(left, right, d_max, levels=None, block=11, alpha=0.9,
                 beta=0.9, sigma_eps=1e-6, sign=MIDDLEBURY, radius=1,
                 workers=1, pyramid=None):
    """matcher.py:398-466. Returns (disparity f64, cost f64, [level dicts]).

    Level dicts carry the counter fields of ``LevelTrace.to_dict`` (no
    wall times), coarsest level first.
    """
    pyr = pyramid if pyramid is not None else build_pyramid(
        left, right, d_max, levels, block)
    trace = []

    def new_tr(k, lv):
        lh, lw = lv[0].shape
        return {"level": k, "height": lh, "width": lw, "d_max": lv[2],
                "block": lv[3], "pixels": lh * lw, "trusted": 0,
                "trusted_evals": 0, "trusted_window_max": 0,
                "full_search_pixels": 0, "selection_evals": 0, "refined": 0,
                "refine_evals": 0, "median_replaced": 0}

    K = len(pyr) - 1
    lv = pyr[K]
    eng = Engine(lv[0], lv[1], lv[3], lv[2], sigma_eps, sign, workers)
    tr = new_tr(K, lv)
    d, c = _process_level(eng, tr, alpha, lambda: match_coarsest(eng))
    tr["full_search_pixels"] = tr["pixels"]
    tr["selection_evals"] = tr["pixels"] * (lv[2] + 1)
    trace.append(tr)
    for k in range(K - 1, -1, -1):
        lv = pyr[k]
        eng = Engine(lv[0], lv[1], lv[3], lv[2], sigma_eps, sign, workers)
        tr = new_tr(k, lv)
        d_hat, c_hat = upsample_prior(d, c, lv[0].shape)
        box = []

        def sel():
            dd, cc, st = select_with_prior(eng, d_hat, c_hat, beta, radius)
            box.append(st)
            return dd, cc

        d, c = _process_level(eng, tr, alpha, sel)
        st = box[0]
        tr["trusted"] = st["trusted"]
        tr["trusted_evals"] = st["trusted_evals"]
        tr["trusted_window_max"] = st["window_max"]
        tr["full_search_pixels"] = st["full_search_pixels"]
        tr["selection_evals"] = st["evals"]
        trace.append(tr)
    return d, c, trace


def total_evals(trace):
    return sum(t["selection_evals"] + t["refine_evals"] for t in trace)


# ---------------------------------------------------------------------------
# SURVEY §8(f) "next" rows: the naive baseline and scoring
# ---------------------------------------------------------------------------

def baseline_bm(left, right, d_max, block, sigma_eps=1e-6, sign="middlebury"):
    """Direct-form full search (baseline.py:18-81): per-block statistics
    from scratch, no box-filter machinery, ties keep the smallest z.
    Vectorised over pixels per disparity (the reference loops per pixel;
    the arithmetic per pixel is the same)."""
    left = np.asarray(left, dtype=np.float64)
    right = np.asarray(right, dtype=np.float64)
    if left.ndim != 2 or left.shape != right.shape:
        raise ValueError("left/right shapes differ")
    if block < 3 or block % 2 == 0:
        raise ValueError("block must be odd and >= 3")
    if d_max < 0:
        raise ValueError("d_max must be >= 0")
    if sign not in ("middlebury", "paper"):
        raise ValueError("unknown sign convention")
    h, w = left.shape
    half = block // 2
    area = block * block
    step = -1 if sign == "middlebury" else 1
    win = np.lib.stride_tricks.sliding_window_view
    lb = win(np.pad(left, half, mode="edge"), (block, block))      # h, w, b, b
    rb = win(np.pad(right, half, mode="edge"), (block, block))
    ldev = lb - lb.mean(axis=(2, 3), keepdims=True)
    lss = (ldev * ldev).sum(axis=(2, 3))
    left_ok = np.sqrt(lss / area) >= sigma_eps
    rdev = rb - rb.mean(axis=(2, 3), keepdims=True)
    rss = (rdev * rdev).sum(axis=(2, 3))
    right_ok = np.sqrt(rss / area) >= sigma_eps
    best_c = np.full((h, w), -2.0)
    best_z = np.zeros((h, w))
    jj = np.arange(w)
    for z in range(d_max + 1):
        col = jj + step * z
        inside = (col >= 0) & (col <= w - 1)
        colc = np.clip(col, 0, w - 1)
        num = (ldev * rdev[:, colc]).sum(axis=(2, 3))
        ok = left_ok & right_ok[:, colc] & inside[None, :]
        with np.errstate(invalid="ignore", divide="ignore"):
            c = np.where(ok, num / np.sqrt(lss * rss[:, colc]), -1.0)
        c = np.minimum(1.0, np.maximum(-1.0, c))
        better = c > best_c
        best_c = np.where(better, c, best_c)
        best_z = np.where(better, float(z), best_z)
    return best_z, best_c, h * w * (d_max + 1)


def evaluate_counts(disparity, gt_values, gt_invalid, scale=1.0,
                    thresholds=(1.0, 2.0, 4.0)):
    """evaluation.py:77-109 as raw counts: (evaluated, [bad counts],
    abs error sum, gt_invalid, output_invalid)."""
    d = np.asarray(disparity, dtype=np.float64)
    out_bad = ~np.isfinite(d)
    gt_bad = np.asarray(gt_invalid, dtype=bool)
    mask = ~out_bad & ~gt_bad
    err = np.abs(d[mask] * scale - np.asarray(gt_values)[mask])
    return (int(mask.sum()), [int((err > t).sum()) for t in thresholds],
            float(err.sum()), int(gt_bad.sum()), int(out_bad.sum()))
