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
