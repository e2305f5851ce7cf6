"""Shared helpers for the test suite (paths, trace packing, parity checker)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

COUNT_KEYS = ("trusted", "trusted_evals", "trusted_window_max",
              "full_search_pixels", "selection_evals", "refined",
              "refine_evals", "median_replaced")


def counts_of(trace):
    """Pack a trace (list of dicts or PipelineTrace) into the golden layout."""
    levels = trace.levels if hasattr(trace, "levels") else trace
    rows = []
    for t in levels:
        t = t if isinstance(t, dict) else t.to_dict()
        rows.append([t["level"], t["height"], t["width"], t["d_max"], t["block"]]
                    + [t[k] for k in COUNT_KEYS])
    return np.array(rows, dtype=np.int64)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def parity_report(d_gpu, c_gpu, d_ref, c_ref, tol=1e-4):
    """SURVEY A.11 parity classification.

    A pixel is *discrepant* when its disparity differs or its cost differs by
    more than ``tol``: both happen only where an fp32-vs-fp64 near-tie flipped
    a winner-take-all or an alpha/beta gate (or downstream of such a flip),
    so discrepant pixels are charged to the 0.05 % budget.  Returns
    (discrepant fraction, max cost error over agreeing disparities excluding
    discrepant pixels, median cost error over all agreeing pixels).
    """
    d_gpu = np.asarray(d_gpu, dtype=np.float64)
    d_ref = np.asarray(d_ref, dtype=np.float64)
    err = np.abs(np.asarray(c_gpu, np.float64) - np.asarray(c_ref, np.float64))
    same = d_gpu == d_ref
    disc = (~same) | (err > tol)
    frac = float(disc.mean())
    ok = ~disc
    cerr = float(err[ok].max()) if ok.any() else 0.0
    med = float(np.median(err[same])) if same.any() else 0.0
    return frac, cerr, med


def counts_close(a, b, rel=2e-3):
    """Trace counters equal, or within ``rel`` when a gate flipped (near-ties)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if np.array_equal(a, b):
        return True
    return bool(np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), 1.0) + 2))


def classify_mismatches(d_gpu, d_ref, left, right, block, d_max, sign="middlebury",
                        tol=1e-4, return_pixels=False, c_gpu=None, alpha=0.9, c_ref=None):
    """Explain level-0 disparity mismatches.

    A mismatch is a *near tie* when the reference's own cost or its clipped
    3x3-averaged cost differs by < ``tol`` between the two disparities, or
    (with ``c_gpu`` / ``c_ref``) when the GPU's or the reference's final cost
    lies within ``tol`` of ``alpha`` (an alpha-gate near tie: refine and
    median run only for C <= alpha; the side that kept the pixel unrefined
    still holds its selection cost, so one of the two maps shows it).  It is
    a *median descendant* when its 5x5 median window holds a near-tie
    mismatch or any alpha-gate near-tie pixel (the gate decides which
    neighbours qualify, matcher.py:345-352).  Returns (n_mismatch, n_near_tie, n_descendant, n_unexplained)
    (+ the unexplained pixels' (row, col) list with ``return_pixels``).
    """
    from oracle import mshbm_oracle as O
    d_gpu = np.asarray(d_gpu).astype(np.int64)
    d_ref = np.asarray(d_ref).astype(np.int64)
    bad = np.argwhere(d_gpu != d_ref)
    if bad.size == 0:
        return (0, 0, 0, 0, []) if return_pixels else (0, 0, 0, 0)
    e = O.Engine(left, right, block, d_max, sign=sign)
    h, w = d_ref.shape
    ties = []
    for i, j in bad:
        a, b = int(d_gpu[i, j]), int(d_ref[i, j])
        own = e.dsi_rows(np.array([i]), np.array([j]))[0]
        nb = [(i + p, j + q) for p in (-1, 0, 1) for q in (-1, 0, 1)
              if 0 <= i + p < h and 0 <= j + q < w]
        s = e.dsi_rows(np.array([r for r, _ in nb]), np.array([c for _, c in nb])).sum(0)
        ties.append(min(abs(own[a] - own[b]), abs(s[a] - s[b]) / len(nb)) < tol)
    ties = np.array(ties)
    gate = np.zeros(d_ref.shape, dtype=bool)
    if c_gpu is not None:
        gate |= np.abs(np.asarray(c_gpu, np.float64) - alpha) < tol
    if c_ref is not None:
        gate |= np.abs(np.asarray(c_ref, np.float64) - alpha) < tol
    ties |= gate[bad[:, 0], bad[:, 1]]
    tie_px = np.concatenate([bad[ties], np.argwhere(gate)])
    desc = 0
    other = []
    for k, (i, j) in enumerate(bad):
        if not ties[k] and tie_px.size and np.any(np.max(np.abs(tie_px - [i, j]), axis=1) <= 2):
            desc += 1
        elif not ties[k]:
            other.append((int(i), int(j)))
    n = len(bad)
    out = (n, int(ties.sum()), desc, n - int(ties.sum()) - desc)
    return out + (other,) if return_pixels else out
