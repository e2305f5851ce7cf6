"""ctypes front of ``libmshbm_oracle.so`` (``oracle/mshbm_oracle.c``) --
TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's CPU leg, tools/).

``run_pipeline`` mirrors ``mshbm_oracle.run_pipeline`` (the numpy
restatement) but streams dense DSI rows per level in C with OpenMP threads,
so full-size BASELINE configs (C3, C5) run in seconds to minutes instead of
hours and fit in host memory.  Counters come back in the golden ``counts``
layout: ``[level, height, width, d_max, block, trusted, trusted_evals,
trusted_window_max, full_search_pixels, selection_evals, refined,
refine_evals, median_replaced]``, coarsest level first.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libmshbm_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "mshbm_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "libmshbm_oracle.so"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.mshbm_oracle_run_pipeline.restype = C.c_int
        L.mshbm_oracle_run_pipeline.argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
            C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
            C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.c_void_p]
        L.mshbm_oracle_match_coarsest.restype = C.c_int
        L.mshbm_oracle_match_coarsest.argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
            C.c_void_p, C.c_void_p]
        L.mshbm_oracle_auto_levels.restype = C.c_int
        L.mshbm_oracle_trace_cols.restype = C.c_int
        _lib = L
    return _lib


def run_pipeline(left, right, d_max, levels=None, block=11, alpha=0.9, beta=0.9,
                 sigma_eps=1e-6, sign="middlebury", radius=1, threads=0, levels_out=False):
    """Returns (disparity f64 (H, W), cost f64 (H, W), counts int64 (K+1, 13)),
    plus, with ``levels_out``, the list of every level's (disparity, cost)
    maps, level 0 first (post-median disparity, refined cost)."""
    L = np.ascontiguousarray(left, dtype=np.float64)
    R = np.ascontiguousarray(right, dtype=np.float64)
    if L.ndim != 2 or L.shape != R.shape:
        raise ValueError(f"left/right shapes differ: {L.shape} vs {R.shape}")
    h, w = L.shape
    lv = -1 if levels is None else int(levels)
    k = lv if lv >= 0 else lib().mshbm_oracle_auto_levels(w, h, int(d_max), int(block))
    d = np.empty((h, w))
    c = np.empty((h, w))
    ncol = lib().mshbm_oracle_trace_cols()
    tr = np.zeros((max(k, 0) + 1, ncol), dtype=np.int64)
    kout = C.c_int(0)
    shapes = [(h, w)]
    for _ in range(max(k, 0)):
        shapes.append(((shapes[-1][0] + 1) // 2, (shapes[-1][1] + 1) // 2))
    tot = sum(a * b for a, b in shapes)
    ld_ = np.empty(tot) if levels_out else None
    lc_ = np.empty(tot) if levels_out else None
    rc = lib().mshbm_oracle_run_pipeline(
        L.ctypes.data, R.ctypes.data, h, w, int(d_max), lv, int(block), int(radius),
        float(alpha), float(beta), float(sigma_eps), 1 if sign == "paper" else 0,
        int(threads), d.ctypes.data, c.ctypes.data, tr.ctypes.data, C.byref(kout),
        ld_.ctypes.data if levels_out else None, lc_.ctypes.data if levels_out else None)
    if rc == 1:
        raise ValueError("invalid pipeline arguments")
    if rc != 0:
        raise MemoryError("oracle out of memory")
    if not levels_out:
        return d, c, tr
    maps, off = [], 0
    for a, b in shapes:
        maps.append((ld_[off:off + a * b].reshape(a, b), lc_[off:off + a * b].reshape(a, b)))
        off += a * b
    return d, c, tr, maps


def match_coarsest(left, right, block, d_max, sigma_eps=1e-6, sign="middlebury"):
    """Full search with first argmax (matcher.py:184-193) -> (d f64, c f64)."""
    L = np.ascontiguousarray(left, dtype=np.float64)
    R = np.ascontiguousarray(right, dtype=np.float64)
    h, w = L.shape
    d = np.empty((h, w))
    c = np.empty((h, w))
    rc = lib().mshbm_oracle_match_coarsest(L.ctypes.data, R.ctypes.data, h, w, int(block),
                                           int(d_max), float(sigma_eps),
                                           1 if sign == "paper" else 0, d.ctypes.data,
                                           c.ctypes.data)
    if rc:
        raise ValueError("invalid engine arguments")
    return d, c
