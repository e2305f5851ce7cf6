"""Next rows of SURVEY §8(f) on the GPU: the naive full-search baseline and
device-side scoring.

* ``baseline_bm`` mirrors ``/root/reference/pkg/src/pyrstereo/baseline.py:18-81``.
  It is an exact single-level full search with no repairs, counting
  H*W*(d_max+1) evaluations.  It runs as the fused sweep through
  ``CostEngine`` + ``match_coarsest``.
* ``evaluate`` / ``compare`` / ``EvalReport`` / ``GroundTruthDisparity`` mirror
  ``evaluation.py:21-123`` and ``formats.py:62-79``.  The metric reduction
  runs on the device (``mshbm_evaluate``), which avoids copying a float64
  disparity map to the host for scoring.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .zncc import SIGN_MIDDLEBURY, SIGN_PAPER_PLUS, CostEngine

__all__ = ["BAD_THRESHOLDS", "GroundTruthDisparity", "EvalReport", "ComparisonSummary",
           "baseline_bm", "evaluate", "compare"]

BAD_THRESHOLDS = (1.0, 2.0, 4.0)


@dataclass
class GroundTruthDisparity:
    """Reference disparities with a per-pixel validity mask (formats.py:62-79)."""

    values: np.ndarray
    invalid: np.ndarray

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]


@dataclass
class EvalReport:
    """Error metrics of one disparity map (evaluation.py:24-63)."""

    bad_1: float
    bad_2: float
    bad_4: float
    avg_abs_err: float
    evaluated: int
    gt_invalid: int
    output_invalid: int
    total_evals: int | None = None
    trust_fractions: tuple | None = None

    _METRICS = ("bad_1", "bad_2", "bad_4", "avg_abs_err", "evaluated", "gt_invalid",
                 "output_invalid")

    def to_dict(self) -> dict:
        """Metrics in report order; effort fields only when set."""
        out = {k: getattr(self, k) for k in self._METRICS}
        if self.total_evals is not None:
            out["total_evals"] = self.total_evals
        if self.trust_fractions is not None:
            out["trust_fractions"] = list(self.trust_fractions)
        return out

    def to_text(self) -> str:
        """``key=value`` lines: floats with 6 decimals, lists comma-joined."""
        def fmt(v):
            if isinstance(v, list):
                return ",".join(f"{x:.6f}" for x in v)
            return f"{v:.6f}" if isinstance(v, float) else str(v)
        return "".join(f"{k}={fmt(v)}\n" for k, v in self.to_dict().items())


@dataclass
class ComparisonSummary:
    """Metric deltas (ours minus reference method) and the effort ratio."""

    deltas: dict = field(default_factory=dict)
    eval_ratio: float | None = None

    def to_dict(self) -> dict:
        return {"deltas": dict(self.deltas), "eval_ratio": self.eval_ratio}


def baseline_bm(left, right, d_max: int, block: int, sigma_eps: float = 1e-6,
                sign: str = SIGN_MIDDLEBURY):
    """Full-search maps plus the evaluation count (baseline.py:18-81)."""
    left = np.asarray(left, dtype=np.float64)
    right = np.asarray(right, dtype=np.float64)
    if left.ndim != 2 or left.shape != right.shape:
        raise ValueError(f"left/right shapes differ: {left.shape} vs {right.shape}")
    if block < 3 or block % 2 == 0:
        raise ValueError(f"block must be odd and >= 3, got {block}")
    if d_max < 0:
        raise ValueError(f"d_max must be >= 0, got {d_max}")
    if sign not in (SIGN_MIDDLEBURY, SIGN_PAPER_PLUS):
        raise ValueError(f"unknown sign convention {sign!r}")
    from .matcher import match_coarsest
    engine = CostEngine(left, right, block, d_max, sigma_eps=sigma_eps, sign=sign)
    d, c = match_coarsest(engine)
    return d, c, engine.counter.count


def evaluate(disparity, gt: GroundTruthDisparity, scale: float = 1.0) -> EvalReport:
    """Score a disparity map against reference disparities (evaluation.py:77-109)."""
    import torch
    d = np.asarray(disparity, dtype=np.float64) if not isinstance(disparity, torch.Tensor) \
        else disparity
    if tuple(d.shape) != tuple(gt.values.shape):
        raise ValueError(f"disparity {tuple(d.shape)} and reference {gt.values.shape} differ")
    if scale <= 0:
        raise ValueError(f"scale must be positive, got {scale}")
    dt = torch.as_tensor(d, dtype=torch.float64).to("cuda").contiguous()
    gv = torch.from_numpy(np.ascontiguousarray(gt.values, dtype=np.float64)).cuda()
    gi = torch.from_numpy(np.ascontiguousarray(gt.invalid, dtype=np.uint8)).cuda()
    taus = (C.c_double * 3)(*BAD_THRESHOLDS)
    counts = (C.c_int64 * 6)()
    abs_sum = C.c_double()
    ctx = _lib.context(dt.device.index)
    _lib.check(_lib.lib().mshbm_evaluate(ctx, dt.data_ptr(), gv.data_ptr(), gi.data_ptr(),
                                         dt.numel(), float(scale), taus, counts,
                                         C.byref(abs_sum), _lib.current_stream()), ctx)
    n = counts[0]
    # same rounding as the reference's 100 * mean(err > tau)
    bad = [100.0 * (counts[k] / n) if n else 0.0 for k in (1, 2, 3)]
    return EvalReport(bad_1=bad[0], bad_2=bad[1], bad_4=bad[2],
                      avg_abs_err=abs_sum.value / n if n else 0.0, evaluated=n,
                      gt_invalid=counts[4], output_invalid=counts[5])


def compare(ours: EvalReport, reference: EvalReport) -> ComparisonSummary:
    """Per-metric deltas plus the ratio of total evaluation counts (evaluation.py:112-123)."""
    deltas = {k: getattr(ours, k) - getattr(reference, k)
              for k in ("bad_1", "bad_2", "bad_4", "avg_abs_err")}
    ratio = None
    if ours.total_evals is not None and reference.total_evals:
        ratio = ours.total_evals / reference.total_evals
    return ComparisonSummary(deltas=deltas, eval_ratio=ratio)
