"""Seeded synthetic stereo workloads for the five BASELINE configurations.

The reference (`pyrstereo`) ships only a constant-shift generator
(`/root/reference/pkg/src/pyrstereo/synthetic.py:37-52`); the BASELINE
configs (`BASELINE.json` "configs") describe a different
one, which is pinned here so that the GPU path, the CPU oracle and the
benchmark all consume the *identical* float32 arrays:

* texture: i.i.d. U[0,1) on the seeded PCG64 stream, Gaussian blur with
  sigma=1.0 (radius 4 = int(4*sigma+0.5), half-sample symmetric borders, the
  scipy ``gaussian_filter`` defaults restated in numpy), min-max stretch to
  [0, 255];
* ground-truth disparity field ``gt[y, x]`` (``_field_*`` below);
* ``right[y, x] = left[y, x + gt[y, x]]`` by linear interpolation along the
  row; samples whose source column leaves the image are filled from an
  independent texture draw;
* i.i.d. N(0, sigma_n^2) noise added to both images; no clipping; float32.

Real Middlebury data is not in this container; these seeded inputs stand in
for it with the shapes, value ranges and disparity ranges the configs state.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["StereoConfig", "CONFIGS", "make_pair", "gaussian_blur", "shifted_pair",
           "interior_mask"]


@dataclass(frozen=True)
class StereoConfig:
    """One BASELINE workload: image geometry, GT model and matching params."""

    name: str
    width: int
    height: int
    field: str                     # "bands" or "planar"
    noise: float                   # sigma_n of the additive noise
    d_max: int                     # full-resolution search bound
    levels: int                    # pyramid halvings K (= stated levels - 1)
    block: int                     # level-0 ZNCC window
    radius: int                    # prior window half-width r
    bands: tuple = ()              # constant-d bands ("bands" field)
    regions: int = 0               # planar regions ("planar" field)
    d_range: tuple = (0.0, 0.0)    # planar disparity range
    seed: int = 0
    batch: int = 1                 # independent pairs (C4)

    @property
    def full_search_pde(self) -> int:
        """W*H*(D+1): the full-search-equivalent (pixel, disparity) count."""
        return self.width * self.height * (self.d_max + 1)


CONFIGS = {
    "C1": StereoConfig("C1", 450, 375, "bands", 2.0, 64, 2, 5, 2,
                       bands=(8.0, 24.0, 48.0), seed=0),
    "C2": StereoConfig("C2", 1472, 992, "bands", 2.0, 144, 3, 7, 2,
                       bands=(10.0, 37.0, 65.0, 92.0, 120.0), seed=1),
    "C3": StereoConfig("C3", 2944, 1984, "planar", 3.0, 288, 4, 9, 3,
                       regions=8, d_range=(0.0, 280.0), seed=2),
    "C4": StereoConfig("C4", 1280, 720, "planar", 2.0, 128, 3, 5, 2,
                       regions=4, d_range=(0.0, 120.0), seed=1000, batch=64),
    "C5": StereoConfig("C5", 8192, 6144, "planar", 8.0, 512, 5, 7, 2,
                       regions=16, d_range=(0.0, 500.0), seed=3),
}


def _gauss_kernel(sigma: float) -> np.ndarray:
    radius = int(4.0 * sigma + 0.5)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def gaussian_blur(img: np.ndarray, sigma: float = 1.0) -> np.ndarray:
    """Separable Gaussian blur, half-sample symmetric borders (float64)."""
    k = _gauss_kernel(sigma)
    r = k.shape[0] // 2
    out = np.asarray(img, dtype=np.float64)
    for axis in (0, 1):
        pad = [(0, 0), (0, 0)]
        pad[axis] = (r, r)
        p = np.pad(out, pad, mode="symmetric")
        acc = np.zeros_like(out)
        n = out.shape[axis]
        for t in range(k.shape[0]):
            sl = [slice(None), slice(None)]
            sl[axis] = slice(t, t + n)
            acc += k[t] * p[tuple(sl)]
        out = acc
    return out


def _texture(rng: np.random.Generator, h: int, w: int) -> np.ndarray:
    t = gaussian_blur(rng.random((h, w)), 1.0)
    lo, hi = t.min(), t.max()
    return (t - lo) * (255.0 / max(hi - lo, 1e-12))


def _field_bands(cfg: StereoConfig, h: int, w: int) -> np.ndarray:
    """Slanted ramp 4 + 0.02 x with equal-width vertical constant bands.

    Band i of n occupies columns [w*(2i+1)/(2n+1), w*(2i+2)/(2n+1)), i.e.
    bands and ramp stripes alternate across the width.
    """
    x = np.arange(w, dtype=np.float64)
    gt = np.broadcast_to(4.0 + 0.02 * x, (h, w)).copy()
    n = len(cfg.bands)
    for i, d in enumerate(cfg.bands):
        x0 = int(w * (2 * i + 1) / (2 * n + 1))
        x1 = int(w * (2 * i + 2) / (2 * n + 1))
        gt[:, x0:x1] = d
    return gt


def _field_planar(cfg: StereoConfig, h: int, w: int,
                  rng: np.random.Generator) -> np.ndarray:
    """Voronoi regions of uniform seeds, each a plane d0 + gx x + gy y.

    d0 ~ U[d_lo, d_hi] at the seed; gradients ~ U[-0.05, 0.05] px/px; the
    field is clipped to [d_lo, d_hi].
    """
    lo, hi = cfg.d_range
    n = cfg.regions
    sy = rng.uniform(0, h, n)
    sx = rng.uniform(0, w, n)
    d0 = rng.uniform(lo, hi, n)
    gx = rng.uniform(-0.05, 0.05, n)
    gy = rng.uniform(-0.05, 0.05, n)
    gt = np.empty((h, w), dtype=np.float64)
    x = np.arange(w, dtype=np.float64)
    for y in range(h):
        d2 = (y - sy[:, None]) ** 2 + (x[None, :] - sx[:, None]) ** 2
        lab = np.argmin(d2, axis=0)
        gt[y] = d0[lab] + gx[lab] * (x - sx[lab]) + gy[lab] * (y - sy[lab])
    return np.clip(gt, lo, hi)


def make_pair(cfg: StereoConfig, seed: int | None = None,
              height: int | None = None, width: int | None = None,
              ) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Build (left, right, gt) float32 arrays for ``cfg`` (optionally resized).

    ``height``/``width`` override the config geometry for parity-size crops
    of a config (same generator, same seed stream, smaller canvas).
    """
    h = cfg.height if height is None else int(height)
    w = cfg.width if width is None else int(width)
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    left = _texture(rng, h, w)
    if cfg.field == "bands":
        gt = _field_bands(cfg, h, w)
    else:
        gt = _field_planar(cfg, h, w, rng)
    fill = _texture(rng, h, w)
    xs = np.arange(w, dtype=np.float64)[None, :] + gt
    x0 = np.floor(xs).astype(np.int64)
    frac = xs - x0
    inside = (x0 >= 0) & (x0 + 1 <= w - 1)
    x0c = np.clip(x0, 0, w - 1)
    x1c = np.clip(x0 + 1, 0, w - 1)
    rows = np.arange(h)[:, None]
    warped = (1.0 - frac) * left[rows, x0c] + frac * left[rows, x1c]
    exact = (x0 == w - 1) & (frac == 0.0)
    right = np.where(inside | exact, warped, fill)
    left = left + rng.normal(0.0, cfg.noise, (h, w))
    right = right + rng.normal(0.0, cfg.noise, (h, w))
    return (left.astype(np.float32), right.astype(np.float32),
            gt.astype(np.float32))


# ---------------------------------------------------------------------------
# Constant-shift fixtures (reference synthetic.py:33-69): band-limited noise
# carved so that right[i, j] == left[i, j + shift] exactly.  Same RNG draws
# as the reference, so seeded pairs are identical.
# ---------------------------------------------------------------------------

def shifted_pair(height: int, width: int, shift: int,
                 rng: np.random.Generator | None = None,
                 cutoff: float = 0.03) -> tuple[np.ndarray, np.ndarray]:
    """Pair whose true disparity is ``shift`` everywhere outside the occluded
    left margin.  ``cutoff`` = maximum spatial frequency (cycles/pixel)."""
    if shift < 0:
        raise ValueError(f"shift must be >= 0, got {shift}")
    if not 0.0 < cutoff <= 0.5:
        raise ValueError(f"cutoff must lie in (0, 0.5], got {cutoff}")
    rng = np.random.default_rng() if rng is None else rng
    cw = width + shift
    noise = rng.standard_normal((height, cw))
    spec = np.fft.rfft2(noise)
    r2 = np.fft.fftfreq(height)[:, None] ** 2 + np.fft.rfftfreq(cw)[None, :] ** 2
    spec[r2 > cutoff * cutoff] = 0.0
    tex = np.fft.irfft2(spec, s=(height, cw))
    lo = tex.min()
    tex = (tex - lo) / max(np.ptp(tex), 1e-12)
    return np.ascontiguousarray(tex[:, :width]), np.ascontiguousarray(tex[:, shift:])


def interior_mask(shape: tuple[int, int], shift: int, block: int,
                  extra: int = 0) -> np.ndarray:
    """Pixels whose block and true match lie inside both images."""
    h, w = shape
    m = block // 2 + extra
    out = np.zeros((h, w), dtype=bool)
    first = max(m + shift, m)
    if h - m > m and w - m > first:
        out[m:h - m, first:w - m] = True
    return out
