"""GPU cost engine (mirror of pyrstereo.zncc).

``CostEngine`` keeps one pyramid level resident on the device
(``mshbm_engine_*`` in the C ABI) and evaluates the reference's ZNCC
(`/root/reference/pkg/src/pyrstereo/zncc.py:144-307`): replicate-padded
b x b windows, -1 for degenerate blocks (sigma < sigma_eps) or right
centres outside the image, clamp to [-1, 1].  Point/row/plane evaluations
run in fp64 (centred); the fused searches (``match_coarsest`` etc.) use the
fp32 sweep kernel.  ``EvalCounter`` counts exactly as the reference's.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = [
    "SIGN_MIDDLEBURY",
    "SIGN_PAPER_PLUS",
    "PatchStats",
    "DsiSlice",
    "EvalCounter",
    "CostEngine",
    "patch_stats",
    "zncc",
    "dsi_entry",
    "averaged_dsi",
]

SIGN_MIDDLEBURY = "middlebury"
SIGN_PAPER_PLUS = "paper"
NEIGHBORHOOD_3X3 = tuple((di, dj) for di in (-1, 0, 1) for dj in (-1, 0, 1))


def sign_code(sign: str) -> int:
    return 1 if sign == SIGN_PAPER_PLUS else 0


@dataclass(frozen=True)
class PatchStats:
    """Mean and RMS deviation of one matching block."""

    mean: float
    sigma: float


@dataclass
class DsiSlice:
    """Costs of one pixel across candidate disparities (zncc.py:68-82)."""

    pixel: tuple[int, int]
    costs: np.ndarray
    evaluated: np.ndarray | None = None

    def __post_init__(self):
        if self.evaluated is None:
            self.evaluated = np.ones(self.costs.shape, dtype=bool)


class EvalCounter:
    """Exact, thread-safe tally of cost evaluations (zncc.py:85-102)."""

    def __init__(self) -> None:
        self._lock = threading.Lock()
        self._count = 0

    def add(self, n: int) -> None:
        with self._lock:
            self._count += int(n)

    @property
    def count(self) -> int:
        return self._count

    def reset(self) -> None:
        with self._lock:
            self._count = 0


def _to_dev(arr, dtype):
    import torch
    if isinstance(arr, torch.Tensor):
        return arr.to(device="cuda", dtype=dtype).contiguous()
    np_dtype = {torch.float64: np.float64, torch.int64: np.int64}[dtype]
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np_dtype)).cuda()


class CostEngine:
    """Disparity-cost evaluator for one pyramid level, resident on the GPU."""

    def __init__(self, left, right, block: int, d_max: int, sigma_eps: float = 1e-6,
                 sign: str = SIGN_MIDDLEBURY, counter: EvalCounter | None = None) -> None:
        import torch
        lt = _to_dev(left, torch.float64)
        rt = _to_dev(right, torch.float64)
        if lt.ndim != 2 or lt.shape != rt.shape:
            raise ValueError(f"left/right shapes differ: {tuple(lt.shape)} vs {tuple(rt.shape)}")
        if block < 3 or block % 2 == 0:
            raise ValueError(f"block must be odd and >= 3, got {block}")
        if d_max < 0:
            raise ValueError(f"d_max must be >= 0, got {d_max}")
        if sign not in (SIGN_MIDDLEBURY, SIGN_PAPER_PLUS):
            raise ValueError(f"unknown sign convention {sign!r}")
        self.height, self.width = int(lt.shape[0]), int(lt.shape[1])
        self.block = int(block)
        self.half = self.block // 2
        self.area = self.block * self.block
        self.d_max = int(d_max)
        self.sigma_eps = float(sigma_eps)
        self.sign = sign
        self.counter = counter if counter is not None else EvalCounter()
        self.device = lt.device
        self._ctx = _lib.context(lt.device.index)
        h = C.c_void_p()
        torch.cuda.current_stream().synchronize()
        _lib.check(_lib.lib().mshbm_engine_create(
            self._ctx, lt.data_ptr(), rt.data_ptr(), self.height, self.width, self.width,
            self.block, self.d_max, self.sigma_eps, sign_code(sign), C.byref(h)), self._ctx)
        self._h = h
        self._stats = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib.lib().mshbm_engine_destroy(h)
            self._h = None

    # -- statistics (zncc.py:185-189), exposed like the reference attributes
    def _load_stats(self):
        if self._stats is None:
            import torch
            t = [torch.empty((self.height, self.width), dtype=torch.float64, device=self.device)
                 for _ in range(4)]
            _lib.check(_lib.lib().mshbm_engine_stats(self._h, *[x.data_ptr() for x in t],
                                                     _lib.current_stream()), self._ctx)
            self._stats = [x.cpu().numpy() for x in t]
        return self._stats

    mean_l = property(lambda self: self._load_stats()[0])
    sigma_l = property(lambda self: self._load_stats()[1])
    mean_r = property(lambda self: self._load_stats()[2])
    sigma_r = property(lambda self: self._load_stats()[3])

    def _check_z(self, z: int) -> int:
        z = int(z)
        if not 0 <= z <= self.d_max:
            raise ValueError(f"disparity {z} outside [0, {self.d_max}]")
        return z

    def plane(self, z: int) -> np.ndarray:
        """Costs of every pixel at one disparity (zncc.py:202-231)."""
        import torch
        z = self._check_z(z)
        out = torch.empty((self.height, self.width), dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().mshbm_engine_plane(self._h, z, out.data_ptr(),
                                                 _lib.current_stream()), self._ctx)
        self.counter.add(self.height * self.width)
        return out.cpu().numpy()

    def full_volume(self, workers: int = 1) -> np.ndarray:
        """All planes stacked as (d_max+1, H, W) (zncc.py:233-249)."""
        return np.stack([self.plane(z) for z in range(self.d_max + 1)])

    def at(self, rows, cols, z) -> np.ndarray:
        """Costs of arbitrary (pixel, disparity) triples (zncc.py:251-269)."""
        import torch
        rows = np.asarray(rows, dtype=np.int64).ravel()
        cols = np.asarray(cols, dtype=np.int64).ravel()
        z = np.asarray(z, dtype=np.int64).ravel()
        if not (rows.shape == cols.shape == z.shape):
            raise ValueError("rows, cols and z must have identical shapes")
        if z.size and (z.min() < 0 or z.max() > self.d_max):
            raise ValueError(f"disparities outside [0, {self.d_max}]")
        n = rows.shape[0]
        if n == 0:
            return np.empty(0)
        rt, ct, zt = (_to_dev(a, torch.int64) for a in (rows, cols, z))
        out = torch.empty(n, dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().mshbm_engine_at(self._h, rt.data_ptr(), ct.data_ptr(),
                                              zt.data_ptr(), n, out.data_ptr(),
                                              _lib.current_stream()), self._ctx)
        self.counter.add(n)
        return out.cpu().numpy()

    def dsi_rows(self, rows, cols) -> np.ndarray:
        """Full cost vectors for a sparse pixel set, shape (S, d_max+1)."""
        import torch
        rows = np.asarray(rows, dtype=np.int64).ravel()
        cols = np.asarray(cols, dtype=np.int64).ravel()
        if rows.shape != cols.shape:
            raise ValueError("rows and cols must have identical shapes")
        n = rows.shape[0]
        out = torch.empty((n, self.d_max + 1), dtype=torch.float64, device=self.device)
        if n:
            rt, ct = _to_dev(rows, torch.int64), _to_dev(cols, torch.int64)
            _lib.check(_lib.lib().mshbm_engine_dsi_rows(self._h, rt.data_ptr(), ct.data_ptr(),
                                                        n, out.data_ptr(),
                                                        _lib.current_stream()), self._ctx)
        self.counter.add(n * (self.d_max + 1))
        return out.cpu().numpy()

    def dsi_slice(self, i: int, j: int) -> DsiSlice:
        costs = self.dsi_rows(np.array([i]), np.array([j]))[0]
        return DsiSlice(pixel=(int(i), int(j)), costs=costs)


def _clipped_patch(img: np.ndarray, i: int, j: int, half: int) -> np.ndarray:
    h, w = img.shape
    if not (0 <= i < h and 0 <= j < w):
        raise ValueError(f"center ({i}, {j}) outside {h}x{w} image")
    rows = np.clip(np.arange(i - half, i + half + 1), 0, h - 1)
    cols = np.clip(np.arange(j - half, j + half + 1), 0, w - 1)
    return img[np.ix_(rows, cols)]


def patch_stats(img, center: tuple[int, int], half: int) -> PatchStats:
    """Mean and RMS deviation of the block around ``center`` (GPU stats kernel)."""
    patch = _clipped_patch(np.asarray(img, dtype=np.float64), center[0], center[1], half)
    e = CostEngine(patch, patch, 2 * half + 1, 0)
    return PatchStats(mean=float(e.mean_l[half, half]), sigma=float(e.sigma_l[half, half]))


def zncc(left, right, center_l: tuple[int, int], center_r: tuple[int, int], half: int,
         sigma_eps: float = 1e-6) -> float:
    """Correlate the blocks around two pixel centres (zncc.py:123-141).

    The two clipped patches become a one-block level pair and are scored by
    the GPU engine at (half, half), z = 0.
    """
    lp = _clipped_patch(np.asarray(left, dtype=np.float64), center_l[0], center_l[1], half)
    rp = _clipped_patch(np.asarray(right, dtype=np.float64), center_r[0], center_r[1], half)
    e = CostEngine(lp, rp, 2 * half + 1, 0, sigma_eps=sigma_eps)
    return float(e.at(np.array([half]), np.array([half]), np.array([0]))[0])


def dsi_entry(engine: CostEngine, i: int, j: int, z: int) -> float:
    """Cost of one pixel at one candidate disparity (zncc.py:322-330)."""
    z = engine._check_z(z)
    return float(engine.at(np.array([i]), np.array([j]), np.array([z]))[0])


def averaged_dsi(engine: CostEngine, i: int, j: int,
                 neighborhood=NEIGHBORHOOD_3X3) -> DsiSlice:
    """Summed cost vector over a pixel's neighborhood (zncc.py:333-350)."""
    coords = [(i + di, j + dj) for di, dj in neighborhood
              if 0 <= i + di < engine.height and 0 <= j + dj < engine.width]
    if not coords:
        return engine.dsi_slice(i, j)
    rows = np.array([c[0] for c in coords])
    cols = np.array([c[1] for c in coords])
    summed = engine.dsi_rows(rows, cols).sum(axis=0)
    return DsiSlice(pixel=(int(i), int(j)), costs=summed)
