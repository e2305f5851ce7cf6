"""Coarse-to-fine block matching on the GPU (mirror of pyrstereo.matcher).

Drop-in for ``/root/reference/pkg/src/pyrstereo/matcher.py``: the same
``MatchConfig`` (plus ``radius``, the prior window half-width the reference
hard-codes to 1 at matcher.py:280,294), the same stage functions and the
same ``run_pipeline(left, right, config, workers=1, pyramid=None) ->
(disparity float64, cost float64, PipelineTrace)``.  All matching runs in
libmshbm.so (sm_100a): ``run_pipeline`` is one C-ABI call that builds the
pyramid, sweeps every level and returns the level-0 maps plus the exact
trace counters; the stage functions call the per-stage entry points.
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .pyramid import StereoPyramid
from .zncc import SIGN_MIDDLEBURY, SIGN_PAPER_PLUS, CostEngine, sign_code

__all__ = [
    "ConfigError",
    "MatchConfig",
    "LevelTrace",
    "PipelineTrace",
    "SelectionStats",
    "match_coarsest",
    "refine_level",
    "upsample_prior",
    "select_with_prior",
    "match_level_with_prior",
    "selective_median",
    "run_pipeline",
    "run_pipeline_device",
    "run_pipeline_band",
    "run_batch",
]

# Launch every kernel directly instead of replaying the plan's CUDA graph
# (tests exercise both paths; stage timings are filled either way, from the
# graph's event-record nodes or the direct path's event records).
DIRECT_LAUNCH = False


def _flags() -> int:
    return _lib.FLAG_TIMING | (_lib.FLAG_NO_GRAPH if DIRECT_LAUNCH else 0)


class ConfigError(ValueError):
    """A matching parameter is outside its legal range."""


@dataclass(frozen=True)
class MatchConfig:
    """Parameters of one matching run (matcher.py:52-84) + ``radius``."""

    d_max: int
    levels: int | None = None
    block: int = 11
    alpha: float = 0.9
    beta: float = 0.9
    sigma_eps: float = 1e-6
    sign: str = SIGN_MIDDLEBURY
    radius: int = 1

    def __post_init__(self) -> None:
        if self.d_max < 1:
            raise ConfigError(f"d_max must be >= 1, got {self.d_max}")
        if self.levels is not None and self.levels < 0:
            raise ConfigError(f"levels must be >= 0, got {self.levels}")
        if self.block < 3 or self.block % 2 == 0:
            raise ConfigError(f"block must be odd and >= 3, got {self.block}")
        if not 0.0 < self.alpha < 1.0:
            raise ConfigError(f"alpha must lie in (0, 1), got {self.alpha}")
        if not 0.0 < self.beta < 1.0:
            raise ConfigError(f"beta must lie in (0, 1), got {self.beta}")
        if self.sigma_eps <= 0.0:
            raise ConfigError(f"sigma_eps must be positive, got {self.sigma_eps}")
        if self.sign not in (SIGN_MIDDLEBURY, SIGN_PAPER_PLUS):
            raise ConfigError(f"unknown sign convention {self.sign!r}")
        if self.radius < 0:
            raise ConfigError(f"radius must be >= 0, got {self.radius}")

    def to_c(self) -> _lib.Config:
        return _lib.Config(d_max=int(self.d_max),
                           levels=-1 if self.levels is None else int(self.levels),
                           block=int(self.block), radius=int(self.radius),
                           alpha=float(self.alpha), beta=float(self.beta),
                           sigma_eps=float(self.sigma_eps), sign=sign_code(self.sign))


@dataclass
class SelectionStats:
    """Bookkeeping of one prior-guided selection pass."""

    trusted: int = 0
    trusted_evals: int = 0
    window_max: int = 0
    full_search_pixels: int = 0
    evals: int = 0


@dataclass
class LevelTrace:
    """Exact per-level counters plus stage wall times (matcher.py:98-153)."""

    level: int
    height: int
    width: int
    d_max: int
    block: int
    trusted: int = 0
    trusted_evals: int = 0
    trusted_window_max: int = 0
    full_search_pixels: int = 0
    selection_evals: int = 0
    refined: int = 0
    refine_evals: int = 0
    median_replaced: int = 0
    seconds: dict = field(default_factory=dict)

    @property
    def pixels(self) -> int:
        return self.height * self.width

    @property
    def trusted_fraction(self) -> float:
        return self.trusted / self.pixels if self.pixels else 0.0

    @property
    def evals(self) -> int:
        return self.selection_evals + self.refine_evals

    def to_dict(self) -> dict:
        return {
            "level": self.level, "height": self.height, "width": self.width,
            "d_max": self.d_max, "block": self.block, "pixels": self.pixels,
            "trusted": self.trusted, "trusted_fraction": self.trusted_fraction,
            "trusted_evals": self.trusted_evals,
            "trusted_window_max": self.trusted_window_max,
            "full_search_pixels": self.full_search_pixels,
            "selection_evals": self.selection_evals, "refined": self.refined,
            "refine_evals": self.refine_evals, "median_replaced": self.median_replaced,
            "seconds": dict(self.seconds),
        }

    @classmethod
    def from_c(cls, t: _lib.LevelTraceC, timed: bool) -> "LevelTrace":
        lt = cls(level=t.level, height=t.height, width=t.width, d_max=t.d_max, block=t.block,
                 trusted=t.trusted, trusted_evals=t.trusted_evals,
                 trusted_window_max=t.trusted_window_max,
                 full_search_pixels=t.full_search_pixels, selection_evals=t.selection_evals,
                 refined=t.refined, refine_evals=t.refine_evals,
                 median_replaced=t.median_replaced)
        if timed:
            # the 3x3-summed refinement runs inside the selection sweep, so
            # its time is reported under "select" and "refine" is 0
            lt.seconds = {"select": t.ms_select / 1e3, "refine": t.ms_refine / 1e3,
                          "median": t.ms_median / 1e3}
            if t.ms_upsample or t.level < 0:
                lt.seconds["upsample"] = t.ms_upsample / 1e3
        return lt


@dataclass
class PipelineTrace:
    """Counters for a full run, coarsest level first (matcher.py:156-181)."""

    levels: list = field(default_factory=list)
    build_seconds: float = 0.0
    total_seconds: float = 0.0

    @property
    def total_evals(self) -> int:
        return sum(lt.evals for lt in self.levels)

    @property
    def trust_fractions(self) -> tuple:
        return tuple(lt.trusted_fraction for lt in self.levels)

    def to_dict(self) -> dict:
        return {"levels": [lt.to_dict() for lt in self.levels],
                "total_evals": self.total_evals, "build_seconds": self.build_seconds,
                "total_seconds": self.total_seconds}

    def counts_dict(self) -> dict:
        out = self.to_dict()
        out.pop("build_seconds")
        out.pop("total_seconds")
        for level in out["levels"]:
            level.pop("seconds")
        return out


# --------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _dev64(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _empty64(shape, device):
    torch = _torch()
    return torch.empty(shape, dtype=torch.float64, device=device)


# --------------------------------------------------------------------- stages
def match_coarsest(engine: CostEngine, workers: int = 1):
    """Full-search disparity and cost maps for one level (matcher.py:184-193)."""
    d = _empty64((engine.height, engine.width), engine.device)
    c = _empty64((engine.height, engine.width), engine.device)
    _lib.check(_lib.lib().mshbm_match_coarsest(engine._h, d.data_ptr(), c.data_ptr(),
                                               _lib.current_stream()), engine._ctx)
    engine.counter.add(engine.height * engine.width * (engine.d_max + 1))
    return d.cpu().numpy(), c.cpu().numpy()


def refine_level(engine: CostEngine, disparity, cost, alpha: float):
    """Re-select low-confidence pixels on 3x3-summed cost vectors (matcher.py:196-233)."""
    dt, ct = _dev64(disparity), _dev64(cost)
    if tuple(ct.shape) != (engine.height, engine.width) or dt.shape != ct.shape:
        raise ValueError("maps must match the level dimensions")
    od, oc = _empty64(ct.shape, ct.device), _empty64(ct.shape, ct.device)
    evals = C.c_int64()
    _lib.check(_lib.lib().mshbm_refine_level(engine._h, dt.data_ptr(), ct.data_ptr(),
                                             float(alpha), od.data_ptr(), oc.data_ptr(),
                                             C.byref(evals), _lib.current_stream()),
               engine._ctx)
    engine.counter.add(evals.value)
    return od.cpu().numpy(), oc.cpu().numpy()


def upsample_prior(d_coarse, c_coarse, target_shape):
    """2x NN disparities, cubic B-spline costs clamped to [-1, 1] (matcher.py:236-260)."""
    h, w = (int(v) for v in target_shape)
    d_coarse = np.asarray(d_coarse, dtype=np.float64)
    c_coarse = np.asarray(c_coarse, dtype=np.float64)
    ch, cw = d_coarse.shape
    if c_coarse.shape != (ch, cw):
        raise ValueError("disparity and cost maps differ in shape")
    if ch != (h + 1) // 2 or cw != (w + 1) // 2:
        raise ValueError(f"{ch}x{cw} maps cannot upsample to {h}x{w}: not the dyadic parent")
    dt, ct = _dev64(d_coarse), _dev64(c_coarse)
    dh, chat = _empty64((h, w), dt.device), _empty64((h, w), dt.device)
    ctx = _lib.context(dt.device.index)
    _lib.check(_lib.lib().mshbm_upsample_prior(ctx, dt.data_ptr(), ct.data_ptr(), ch, cw, h, w,
                                               dh.data_ptr(), chat.data_ptr(),
                                               _lib.current_stream()), ctx)
    return dh.cpu().numpy(), chat.cpu().numpy()


def select_with_prior(engine: CostEngine, d_hat, c_hat, beta: float, radius: int = 1):
    """Prior-guided selection (matcher.py:263-320), window +-radius."""
    dt, ct = _dev64(d_hat), _dev64(c_hat)
    h, w = ct.shape
    if tuple(dt.shape) != (h, w) or (engine.height, engine.width) != (h, w):
        raise ValueError("prior maps must match the level dimensions")
    od, oc = _empty64((h, w), ct.device), _empty64((h, w), ct.device)
    st = (C.c_int64 * 5)()
    _lib.check(_lib.lib().mshbm_select_with_prior(engine._h, dt.data_ptr(), ct.data_ptr(),
                                                  float(beta), int(radius), od.data_ptr(),
                                                  oc.data_ptr(), st, _lib.current_stream()),
               engine._ctx)
    stats = SelectionStats(trusted=st[0], trusted_evals=st[1], window_max=st[2],
                           full_search_pixels=st[3], evals=st[4])
    engine.counter.add(stats.evals)
    return od.cpu().numpy(), oc.cpu().numpy(), stats


def selective_median(disparity, cost, alpha: float) -> np.ndarray:
    """Lower median of confident 5x5 neighbours for low-cost pixels (matcher.py:323-359)."""
    dt, ct = _dev64(disparity), _dev64(cost)
    if dt.shape != ct.shape:
        raise ValueError("disparity and cost maps differ in shape")
    h, w = ct.shape
    out = _empty64((h, w), ct.device)
    ctx = _lib.context(ct.device.index)
    _lib.check(_lib.lib().mshbm_selective_median(ctx, dt.data_ptr(), ct.data_ptr(), h, w,
                                                 float(alpha), out.data_ptr(), None,
                                                 _lib.current_stream()), ctx)
    return out.cpu().numpy()


def match_level_with_prior(engine: CostEngine, d_hat, c_hat, alpha: float, beta: float,
                           radius: int = 1):
    """select -> refine -> median for one finer level (matcher.py:362-369)."""
    disparity, cost, _ = select_with_prior(engine, d_hat, c_hat, beta, radius)
    disparity, cost = refine_level(engine, disparity, cost, alpha)
    disparity = selective_median(disparity, cost, alpha)
    return disparity, cost


# --------------------------------------------------------------------- pipeline
def _as_f32(img) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(img, dtype=np.float64).astype(np.float32)
                                if np.asarray(img).dtype != np.float32 else img,
                                dtype=np.float32)


def _trace_from(tr, K: int, timed: bool, t_start: float, user_pyramid: bool = False
                ) -> PipelineTrace:
    """PipelineTrace from the C records; build_seconds is the device time of
    the pyramid construction (0 for a caller-supplied pyramid, as the
    reference, matcher.py:410-416)."""
    build = 0.0 if (user_pyramid or not timed) else tr[0].ms_build / 1e3
    out = PipelineTrace(build_seconds=build)
    out.levels = [LevelTrace.from_c(tr[t], timed) for t in range(K + 1)]
    out.total_seconds = time.perf_counter() - t_start
    return out


def run_pipeline(left, right, config: MatchConfig, workers: int = 1,
                 pyramid: StereoPyramid | None = None):
    """Full-resolution disparity and cost maps for a pair (matcher.py:398-466).

    Returns ``(disparity, cost, trace)`` as the reference: float64 (H, W)
    maps (integer-valued disparities) and a ``PipelineTrace`` with exact
    counters, coarsest level first.  ``workers`` is accepted and ignored.
    """
    t_start = time.perf_counter()
    if pyramid is not None:
        return _run_user_pyramid(pyramid, config, t_start)
    lf = np.asarray(left)
    rf = np.asarray(right)
    if lf.ndim != 2 or lf.shape != rf.shape:
        raise ValueError(f"left/right shapes differ: {lf.shape} vs {rf.shape}")
    h, w = lf.shape
    cfg = config.to_c()
    K = C.c_int32()
    ctx = _lib.context()
    _lib.check(_lib.lib().mshbm_resolve_levels(C.byref(cfg), h, w, C.byref(K)))
    tr = (_lib.LevelTraceC * (K.value + 1))()
    with _PIN_LOCK:
        pl, pr, pd, pc = _pinned(h, w)
        _stage_f32(pl, lf)
        _stage_f32(pr, rf)
        _lib.check(_lib.lib().mshbm_run_pipeline(
            ctx, pl.data_ptr(), pr.data_ptr(), h, w, w, C.byref(cfg), pd.data_ptr(),
            pc.data_ptr(), w, tr, C.byref(K), _lib.IO_HOST, _flags(), None), ctx)
        torch = _torch()
        disparity = pd.to(torch.float64).numpy()
        cost = pc.to(torch.float64).numpy()
    trace = _trace_from(tr, K.value, True, t_start)
    return disparity, cost, trace


# Host staging of the drop-in: page-locked buffers per image shape (the
# copies to and from the device then run at PCIe rate instead of through the
# driver's pageable path), filled and converted by torch's threaded CPU
# copies: float32 <- the caller's array (any dtype, rounded as
# asarray(float64).astype(float32)), fresh float64 maps <- int16 / float32.
_PIN: dict = {}
_PIN_LOCK = threading.Lock()


def _pinned(h: int, w: int):
    torch = _torch()
    buf = _PIN.get((h, w))
    if buf is None:
        if len(_PIN) >= 4:
            _PIN.clear()
        buf = (torch.empty((h, w), dtype=torch.float32).pin_memory(),
               torch.empty((h, w), dtype=torch.float32).pin_memory(),
               torch.empty((h, w), dtype=torch.int16).pin_memory(),
               torch.empty((h, w), dtype=torch.float32).pin_memory())
        _PIN[(h, w)] = buf
    return buf


def _stage_f32(dst, img: np.ndarray) -> None:
    torch = _torch()
    if img.dtype not in (np.float32, np.float64):
        img = _as_f32(img)
    elif not img.flags.c_contiguous:
        img = np.ascontiguousarray(img)
    if not img.flags.writeable:      # torch.from_numpy warns on read-only arrays
        img = img.copy()
    dst.copy_(torch.from_numpy(img))


def run_pipeline_device(left, right, config: MatchConfig, trace: bool = True, stream=None):
    """GPU-resident variant: torch CUDA float32 inputs -> (int16, float32) CUDA maps.

    Asynchronous on ``stream`` (default: torch's current stream) when
    ``trace`` is False; with ``trace`` it synchronises to read the counters.
    """
    torch = _torch()
    lt = left.to(device="cuda", dtype=torch.float32).contiguous()
    rt = right.to(device="cuda", dtype=torch.float32).contiguous()
    if lt.ndim != 2 or lt.shape != rt.shape:
        raise ValueError(f"left/right shapes differ: {tuple(lt.shape)} vs {tuple(rt.shape)}")
    h, w = lt.shape
    cfg = config.to_c()
    K = C.c_int32()
    ctx = _lib.context(lt.device.index)
    _lib.check(_lib.lib().mshbm_resolve_levels(C.byref(cfg), h, w, C.byref(K)))
    d16 = torch.empty((h, w), dtype=torch.int16, device=lt.device)
    c32 = torch.empty((h, w), dtype=torch.float32, device=lt.device)
    tr = (_lib.LevelTraceC * (K.value + 1))() if trace else None
    s = C.c_void_p(stream.cuda_stream) if stream is not None else _lib.current_stream()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().mshbm_run_pipeline(
        ctx, lt.data_ptr(), rt.data_ptr(), h, w, w, C.byref(cfg), d16.data_ptr(),
        c32.data_ptr(), w, tr, C.byref(K), _lib.IO_DEVICE, _flags() if trace else 0, s), ctx)
    t = _trace_from(tr, K.value, True, t0) if trace else None
    return d16, c32, t


def _run_user_pyramid(pyramid: StereoPyramid, config: MatchConfig, t_start: float):
    """run_pipeline(..., pyramid=...) (matcher.py:410-416): levels used as given."""
    torch = _torch()
    n = len(pyramid)
    L = [_dev64(lv.left) for lv in pyramid.levels]
    R = [_dev64(lv.right) for lv in pyramid.levels]
    for a, b in zip(L, R):
        if a.ndim != 2 or a.shape != b.shape:
            raise ValueError("pyramid level left/right shapes differ")
    arr = lambda t, v: (t * n)(*v)  # noqa: E731
    ptrL = arr(C.c_void_p, [t.data_ptr() for t in L])
    ptrR = arr(C.c_void_p, [t.data_ptr() for t in R])
    hs = arr(C.c_int32, [t.shape[0] for t in L])
    ws = arr(C.c_int32, [t.shape[1] for t in L])
    lds = arr(C.c_int64, [t.shape[1] for t in L])
    dms = arr(C.c_int32, [lv.d_max for lv in pyramid.levels])
    bks = arr(C.c_int32, [lv.block for lv in pyramid.levels])
    cfg = config.to_c()
    h, w = L[0].shape
    d16 = torch.empty((h, w), dtype=torch.int16, device=L[0].device)
    c32 = torch.empty((h, w), dtype=torch.float32, device=L[0].device)
    tr = (_lib.LevelTraceC * n)()
    ctx = _lib.context(L[0].device.index)
    _lib.check(_lib.lib().mshbm_run_pyramid(ctx, n, ptrL, ptrR, hs, ws, lds, dms, bks,
                                            C.byref(cfg), d16.data_ptr(), c32.data_ptr(), w,
                                            tr, _lib.current_stream()), ctx)
    trace = _trace_from(tr, n - 1, False, t_start, user_pyramid=True)
    return (d16.cpu().numpy().astype(np.float64), c32.cpu().numpy().astype(np.float64), trace)


# --------------------------------------------------------------------- C4 / C5
def run_batch(lefts, rights, config: MatchConfig, n_streams: int = 4, trace: bool = True):
    """Independent same-shape pairs (BASELINE C4) through ``mshbm_run_batch``.

    ``lefts``/``rights``: a stacked torch CUDA tensor (N, H, W) or a sequence
    of arrays.  Pairs run round-robin on ``n_streams`` concurrent CUDA-graph
    plans.  Returns (disparities int16 (N, H, W), costs float32 (N, H, W),
    traces | None) as CUDA tensors.
    """
    torch = _torch()
    L = torch.stack([torch.as_tensor(x) for x in lefts]) if not isinstance(lefts, torch.Tensor) else lefts
    R = torch.stack([torch.as_tensor(x) for x in rights]) if not isinstance(rights, torch.Tensor) else rights
    L = L.to(device="cuda", dtype=torch.float32).contiguous()
    R = R.to(device="cuda", dtype=torch.float32).contiguous()
    if L.ndim != 3 or L.shape != R.shape:
        raise ValueError(f"batch shapes differ: {tuple(L.shape)} vs {tuple(R.shape)}")
    n, h, w = L.shape
    cfg = config.to_c()
    K = C.c_int32()
    _lib.check(_lib.lib().mshbm_resolve_levels(C.byref(cfg), h, w, C.byref(K)))
    D = torch.empty((n, h, w), dtype=torch.int16, device=L.device)
    Cc = torch.empty((n, h, w), dtype=torch.float32, device=L.device)
    ptrs = lambda t: (C.c_void_p * n)(*[t[i].data_ptr() for i in range(n)])  # noqa: E731
    tr = (_lib.LevelTraceC * (n * (K.value + 1)))() if trace else None
    ctx = _lib.context(L.device.index)
    _lib.check(_lib.lib().mshbm_run_batch(ctx, n, ptrs(L), ptrs(R), h, w, w, C.byref(cfg),
                                          ptrs(D), ptrs(Cc), w, tr, _lib.IO_DEVICE,
                                          int(n_streams), _lib.current_stream()), ctx)
    traces = None
    if trace:
        k1 = K.value + 1
        traces = []
        for i in range(n):
            t = PipelineTrace()
            t.levels = [LevelTrace.from_c(tr[i * k1 + l], False) for l in range(k1)]
            traces.append(t)
    return D, Cc, traces


def run_pipeline_band(left, right, config: MatchConfig, row_begin: int, row_end: int,
                      trace: bool = True, timed: bool = False):
    """Level-0 rows [row_begin, row_end) of run_pipeline (BASELINE C5 bands).

    Bit-identical to the same rows of the whole-image result; limits must be
    multiples of 2^levels (or the image height).  Trace counters cover the
    band's own rows at every level, so a partition's traces sum to the
    whole-image trace (see ``sharding.merge_traces``).  CUDA tensors in/out.
    """
    torch = _torch()
    lt = left.to(device="cuda", dtype=torch.float32).contiguous()
    rt = right.to(device="cuda", dtype=torch.float32).contiguous()
    if lt.ndim != 2 or lt.shape != rt.shape:
        raise ValueError(f"left/right shapes differ: {tuple(lt.shape)} vs {tuple(rt.shape)}")
    h, w = lt.shape
    cfg = config.to_c()
    K = C.c_int32()
    ctx = _lib.context(lt.device.index)
    n = int(row_end) - int(row_begin)
    d16 = torch.empty((max(n, 0), w), dtype=torch.int16, device=lt.device)
    c32 = torch.empty((max(n, 0), w), dtype=torch.float32, device=lt.device)
    _lib.check(_lib.lib().mshbm_resolve_levels(C.byref(cfg), h, w, C.byref(K)))
    tr = (_lib.LevelTraceC * (K.value + 1))() if trace else None
    _lib.check(_lib.lib().mshbm_run_pipeline_band(
        ctx, lt.data_ptr(), rt.data_ptr(), h, w, w, C.byref(cfg), int(row_begin), int(row_end),
        d16.data_ptr(), c32.data_ptr(), w, tr, C.byref(K), _lib.IO_DEVICE,
        _lib.FLAG_TIMING if (trace and timed) else 0, _lib.current_stream()), ctx)
    t = _trace_from(tr, K.value, trace and timed, time.perf_counter()) if trace else None
    return d16, c32, t
