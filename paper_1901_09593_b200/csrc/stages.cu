// HBM-bound stage kernels: pyramid (K1), window statistics (K2), cubic
// B-spline prior (K5), selective median (K4), and the CostEngine / stage-API
// helpers (direct fp64 evaluation, gate combines).
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mshbm {

namespace {

constexpr unsigned kFull = 0xffffffffu;

inline dim3 grid2d(int w, int h, dim3 blk, int z = 1) {
  return dim3((w + blk.x - 1) / blk.x, (h + blk.y - 1) / blk.y, z);
}

// ------------------------------------------------------------------ K1
__global__ void f32_to_f64_kernel(const float* a, const float* b, int h, int w,
                                  int64_t ldi, double* oa, double* ob,
                                  int64_t ldo) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const float* src = blockIdx.z ? b : a;
  double* dst = blockIdx.z ? ob : oa;
  dst[(int64_t)y * ldo + x] = (double)src[(int64_t)y * ldi + x];
}

// gaussian_downsample (pyramid.py:65-81): (1,4,6,4,1)/16 along axis 0, then
// axis 1, replicate borders, keep even rows/cols.  Only the kept samples are
// computed: out(I,J) = sum_b k_b sum_a k_a X(2I+a-2, 2J+b-2) (clamped).
// COPY: level 0 from the fp32 input -- the same kernel also writes the exact
// fp64 copy of its 2x2 input block (the level-0 image), so the pipeline needs
// no separate conversion pass.
template <typename T, bool COPY>
__global__ void downsample_kernel(const T* in0, const T* in1, int h, int w, int64_t ldi,
                                  double* out0, double* out1, int64_t ldo, int oh, int ow,
                                  double* cp0, double* cp1, int64_t ldc, int i0, int i1,
                                  int step) {
  pdl_wait();
  // output rows [i0, i1) only (row bands compute the rows their levels need)
  const int J = blockIdx.x * blockDim.x + threadIdx.x;
  const int I = i0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (J >= ow || I >= oh || I >= i1) return;
  const T* in = blockIdx.z ? in1 : in0;
  double* out = blockIdx.z ? out1 : out0;
  const double k[5] = {1.0 / 16.0, 4.0 / 16.0, 6.0 / 16.0, 4.0 / 16.0, 1.0 / 16.0};
  int rows[5];
#pragma unroll
  for (int a = 0; a < 5; ++a) rows[a] = clampi(step * I + a - 2, 0, h - 1);
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int col = clampi(step * J + b - 2, 0, w - 1);
    double v = 0.0;
#pragma unroll
    for (int a = 0; a < 5; ++a) v += k[a] * (double)in[(int64_t)rows[a] * ldi + col];
    acc += k[b] * v;
  }
  out[(int64_t)I * ldo + J] = acc;
  if constexpr (COPY) {
    double* cp = blockIdx.z ? cp1 : cp0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int y = 2 * I + a, x = 2 * J + b;
        if (y < h && x < w) cp[(int64_t)y * ldc + x] = (double)in[(int64_t)y * ldi + x];
      }
  }
}

// gaussian_downsample, pipeline form: a 32 x 16 output tile per CTA.  The
// replicate-clamped input region (35 x 67) is staged in shared memory with
// coalesced row loads, then the vertical 5-tap pass (only the kept rows)
// and the horizontal pass (only the kept columns) -- the same arithmetic
// and order as downsample_kernel, so the values are identical.
template <typename T>
__global__ void __launch_bounds__(256) downsample_tile_kernel(const T* in0, const T* in1, int h,
                                                              int w, int64_t ldi, double* out0,
                                                              double* out1, int64_t ldo, int oh,
                                                              int ow, int i0, int i1) {
  pdl_wait();
  constexpr int OW = 32, OH = 16, IR = 2 * OH + 3, IC = 2 * OW + 3;
  __shared__ double X[IR][IC];
  // kept columns 2J + b in two planes by parity: Ve[I][m] = column 2m,
  // Vo[I][m] = column 2m + 1, so the horizontal pass reads consecutive
  // doubles across lanes
  __shared__ double Ve[OH][OW + 2], Vo[OH][OW + 2];
  const T* in = blockIdx.z ? in1 : in0;
  double* out = blockIdx.z ? out1 : out0;
  const int J0 = blockIdx.x * OW, I0 = i0 + blockIdx.y * OH;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8, no index divisions
  {
    // every load of the thread in flight before the shared-memory stores
    constexpr int NRW = (IR + 7) / 8, NCL = (IC + 31) / 32;
    T v[NRW][NCL];
    int xc[NCL];
#pragma unroll
    for (int q = 0; q < NCL; ++q) xc[q] = clampi(2 * J0 - 2 + tx + 32 * q, 0, w - 1);
#pragma unroll
    for (int p = 0; p < NRW; ++p) {
      const int r = ty + 8 * p;
      const T* row = in + (int64_t)clampi(2 * I0 - 2 + r, 0, h - 1) * ldi;
#pragma unroll
      for (int q = 0; q < NCL; ++q)
        if (r < IR && tx + 32 * q < IC) v[p][q] = row[xc[q]];
    }
#pragma unroll
    for (int p = 0; p < NRW; ++p)
#pragma unroll
      for (int q = 0; q < NCL; ++q) {
        const int r = ty + 8 * p, c = tx + 32 * q;
        if (r < IR && c < IC) X[r][c] = (double)v[p][q];
      }
  }
  __syncthreads();
  const double k[5] = {1.0 / 16.0, 4.0 / 16.0, 6.0 / 16.0, 4.0 / 16.0, 1.0 / 16.0};
  for (int I = ty; I < OH; I += 8) {
    for (int c = tx; c < IC; c += 32) {
      double v = 0.0;
#pragma unroll
      for (int a = 0; a < 5; ++a) v += k[a] * X[2 * I + a][c];
      if (c & 1) Vo[I][c >> 1] = v;
      else Ve[I][c >> 1] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < OH / 8; ++q) {
    const int I = ty + 8 * q, J = tx;
    const int gi = I0 + I, gj = J0 + J;
    if (gi >= i1 || gi >= oh || gj >= ow) continue;
    // columns 2J .. 2J + 4 = Ve[J], Vo[J], Ve[J + 1], Vo[J + 1], Ve[J + 2]
    double acc = 0.0;
    acc += k[0] * Ve[I][J];
    acc += k[1] * Vo[I][J];
    acc += k[2] * Ve[I][J + 1];
    acc += k[3] * Vo[I][J + 1];
    acc += k[4] * Ve[I][J + 2];
    out[(int64_t)gi * ldo + gj] = acc;
  }
}

// ------------------------------------------------------------------ K2
// Box mean and centred sigma of the b x b replicate-padded window
// (zncc.py:185-189 computes the same quantities via uniform_filter raw
// moments; centred arithmetic keeps flat patches at sigma == 0 exactly).
template <bool F64>
__global__ void stats_kernel(const double* img, int h, int w, int64_t ld,
                             int b, double sigma_eps, float* mu32, float* is32,
                             double* mu64, double* sg64, int64_t lds, int y_base = 0) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = y_base + blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const int h2 = b / 2;
  double s = 0.0;
  for (int r = 0; r < b; ++r) {
    const double* row = img + (int64_t)clampi(y + r - h2, 0, h - 1) * ld;
    for (int c = 0; c < b; ++c) s += row[clampi(x + c - h2, 0, w - 1)];
  }
  const double area = (double)(b * b);
  const double mu = s / area;
  double ss = 0.0;
  for (int r = 0; r < b; ++r) {
    const double* row = img + (int64_t)clampi(y + r - h2, 0, h - 1) * ld;
    for (int c = 0; c < b; ++c) {
      const double dv = row[clampi(x + c - h2, 0, w - 1)] - mu;
      ss += dv * dv;
    }
  }
  const double sigma = sqrt(ss / area);
  if (F64) {
    mu64[(int64_t)y * w + x] = mu;
    sg64[(int64_t)y * w + x] = sigma;
  } else {
    mu32[(int64_t)y * lds + x] = (float)mu;
    is32[(int64_t)y * lds + x] = sigma >= sigma_eps ? (float)(1.0 / sigma) : 0.f;
  }
}

// ------------------------------------------------------------------ K5
// scipy map_coordinates(order=3, mode='nearest') (matcher.py:259):
// _prepad_for_spline_filter pads 12 samples by edge replication, then
// spline_filter1d along axis 0 and axis 1 with the cubic pole
// z = sqrt(3) - 2, gain (1-z)(1-1/z), 'reflect' causal/anticausal init.
constexpr int kNpad = 12;

constexpr double kPole = -0.26794919243112270;   // sqrt(3) - 2

// The prefilter as a parallel FIR.  scipy's recursion (gain (1-z)(1-1/z),
// causal + anticausal pass, exact 'reflect' initialisation at both line
// ends) equals, on each axis, the symmetric filter h[m] = sqrt(3) z^|m|
// applied to the half-sample-symmetric periodic extension of the padded
// line (checked against the recursion to 1e-15 in tests).  |z|^29 < 3e-17,
// so taps |m| <= 28 reproduce it to fp64 rounding.  Every output is an
// independent 57-tap dot product: no sequential recursion, and a row band's
// coefficients depend only on the +-28 padded rows around them.
constexpr int kFirR = 28;
constexpr int kFT = 32;                    // output tile (padded coords)
constexpr int kFE = kFT + 2 * kFirR;       // 88: staged region per axis

__device__ __forceinline__ double fir_tap(int m) {
  // sqrt(3) * z^m, m in [0, 28], by repeated multiplication at compile time
  double t = 1.7320508075688772;
#pragma unroll
  for (int k = 0; k < 28; ++k)
    if (k < m) t *= kPole;
  return t;
}

// half-sample-symmetric periodic extension of an index into [0, n)
__device__ __forceinline__ int reflect_index(int p, int n) {
  if (p >= 0 && p < n) return p;                 // interior: no division
  if (p < 0 && p >= -n) return -1 - p;
  if (p >= n && p < 2 * n) return 2 * n - 1 - p;
  const int per = 2 * n;
  int q = p % per;
  if (q < 0) q += per;
  return q < n ? q : per - 1 - q;
}

template <typename T>
__global__ void __launch_bounds__(256) bspline_fir_kernel(const T* cin, int ch, int cw,
                                                          int64_t ldcin, double* coef,
                                                          int64_t ldc, int ty0) {
  extern __shared__ double smem_d[];
  T (*S)[kFE + 1] = reinterpret_cast<T (*)[kFE + 1]>(smem_d);        // [kFE][kFE+1] input
  // axis-0 pass [kFT][kFE]: a pitch of 88 doubles (= 16 words mod 32) puts the
  // axis-1 reads of a warp (4 rows x 8 consecutive doubles) on 2 x 32 banks
  double (*Tm)[kFE] = reinterpret_cast<double (*)[kFE]>(
      smem_d + (sizeof(T) * kFE * (kFE + 1) + 7) / 8);
  const int nh = ch + 2 * kNpad, nw = cw + 2 * kNpad;
  // tile rows ty0.. (row bands: only the coefficient rows their prior reads)
  const int y0 = (ty0 + blockIdx.y) * kFT, x0 = blockIdx.x * kFT;
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 warps
  // stage the doubly extended padded input: P[y][x] = cost[clamp(y-12)][clamp(x-12)].
  // All of a thread's loads are issued before any store, so their latency
  // overlaps (a load->store loop would serialise ~31 memory round trips).
  {
    constexpr int kPer = (kFE * kFE + 255) / 256;   // 31
    T v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = threadIdx.x + 256 * k;
      const int r = t / kFE, c = t - r * kFE;
      const int py = reflect_index(y0 - kFirR + r, nh);
      const int px = reflect_index(x0 - kFirR + c, nw);
      v[k] = t < kFE * kFE ? cin[(int64_t)clampi(py - kNpad, 0, ch - 1) * ldcin +
                                  clampi(px - kNpad, 0, cw - 1)]
                           : T(0);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = threadIdx.x + 256 * k;
      const int r = t / kFE, c = t - r * kFE;
      if (t < kFE * kFE) S[r][c] = v[k];
    }
  }
  __syncthreads();
  // axis 0: rows ty, ty+8, ty+16, ty+24 of the tile share the staged rows
  for (int c = lane; c < kFE; c += 32) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 2 * kFirR + 1 + 24; ++k) {
      const double v = (double)S[ty + k][c];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int m = k - 8 * o - kFirR;
        if (m >= -kFirR && m <= kFirR) acc[o] = fma(fir_tap(m < 0 ? -m : m), v, acc[o]);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) Tm[ty + 8 * o][c] = acc[o];
  }
  __syncthreads();
  // axis 1: thread (row r, q) computes columns q, q + 8, q + 16, q + 24 of
  // its row from the 81 row samples they share (the same tap order per
  // output as a 57-tap loop: m ascending)
  {
    const int r = threadIdx.x >> 3, q = threadIdx.x & 7;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 2 * kFirR + 1 + 24; ++k) {
      const double v = Tm[r][q + k];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int m = k - 8 * o - kFirR;
        if (m >= -kFirR && m <= kFirR) acc[o] = fma(fir_tap(m < 0 ? -m : m), v, acc[o]);
      }
    }
    const int gy = y0 + r;
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int gx = x0 + q + 8 * o;
      if (gy < nh && gx < nw) coef[(int64_t)gy * ldc + gx] = acc[o];
    }
  }
}

__device__ __forceinline__ void bspline_w(double t, double* wgt) {
  constexpr double k6 = 1.0 / 6.0;   // multiply: fp64 division is a subroutine call
  const double u = 1.0 - t, t2 = t * t, t3 = t2 * t;
  wgt[0] = u * u * u * k6;
  wgt[1] = (4.0 - 6.0 * t2 + 3.0 * t3) * k6;
  wgt[2] = (1.0 + 3.0 * t + 3.0 * t2 - 3.0 * t3) * k6;
  wgt[3] = t3 * k6;
}

// spline value at fine pixel (i, j) of an h x w target from a ch x cw map
__device__ double spline_at(const double* coef, int64_t ldc, int ch, int cw,
                            int h, int w, int i, int j) {
  const double y = ((double)i + 0.5) * ((double)ch / (double)h) - 0.5 + kNpad;
  const double x = ((double)j + 0.5) * ((double)cw / (double)w) - 0.5 + kNpad;
  const double fy = floor(y), fx = floor(x);
  double wy[4], wx[4];
  bspline_w(y - fy, wy);
  bspline_w(x - fx, wx);
  const int iy = (int)fy - 1, ix = (int)fx - 1;
  const int nh = ch + 2 * kNpad, nw = cw + 2 * kNpad;
  double out = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* row = coef + (int64_t)clampi(iy + a, 0, nh - 1) * ldc;
    double r = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) r += wx[b] * row[clampi(ix + b, 0, nw - 1)];
    out += wy[a] * r;
  }
  return out;
}

// Trace counters of select_with_prior (matcher.py:288-308, A.10):
// trusted, sum of legal window sizes, max window size.
__device__ __forceinline__ void count_trusted(bool trusted, int c, int r, int d,
                                              unsigned long long* counters) {
  long long ws = 0;
  if (trusted) ws = (long long)(min(c + r, d) - max(c - r, 0) + 1);
  const int slot[3] = {kCntTrusted, kCntTrustedEvals, kCntWindowMax};
  const unsigned long long val[3] = {trusted ? 1ull : 0ull, (unsigned long long)ws,
                                     (unsigned long long)ws};
  const bool mx[3] = {false, false, true};
  block_accumulate<3>(counters, slot, val, mx);
}

__global__ void prior_maps_kernel(const double* d_hat, const double* c_hat,
                                  int h, int w, int d, int r, double beta,
                                  int* wc, int64_t ldw,
                                  unsigned long long* counters) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const bool in = i < h && j < w;
  bool trusted = false;
  int center = 0;
  if (in) {
    const double dh = d_hat[(int64_t)i * w + j];
    const bool finite = isfinite(dh);
    const double cen = finite ? trunc(dh) : 0.0;     // astype(np.intp)
    const bool ok = finite && (cen + r >= 0.0) && (cen - r <= (double)d);
    trusted = (c_hat[(int64_t)i * w + j] > beta) && ok;
    center = trusted ? (int)cen : 0;
    wc[(int64_t)i * ldw + j] = trusted ? center : kWcNone;
  }
  count_trusted(trusted, center, r, d, counters);
}

__global__ void upsample_kernel(const double* dco, int ch, int cw,
                                const double* coef, int64_t ldc, int h, int w,
                                double* d_hat, double* c_hat) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= h || j >= w) return;
  const double c = spline_at(coef, ldc, ch, cw, h, w, i, j);
  c_hat[(int64_t)i * w + j] = fmin(fmax(c, -1.0), 1.0);
  d_hat[(int64_t)i * w + j] = 2.0 * dco[(int64_t)(i >> 1) * cw + (j >> 1)];
}

// ------------------------------------------------------------------ K4
// selective_median (matcher.py:323-359): a pixel with C <= alpha takes the
// lower median of the disparities in its clipped 5x5 window whose own
// cost exceeds alpha (and are finite); none -> unchanged.
template <typename T>
__device__ __forceinline__ T lower_median(T* v, int n) {
  const int m = (n - 1) >> 1;
  T best = v[0];
  for (int k = 0; k < n; ++k) {
    int less = 0, leq = 0;
    for (int t = 0; t < n; ++t) {
      less += v[t] < v[k];
      leq += v[t] <= v[k];
    }
    if (less <= m && m < leq) { best = v[k]; break; }
  }
  return best;
}

__global__ void median_f64_kernel(const double* d, const double* c, int h,
                                  int w, double alpha, double* out,
                                  unsigned long long* replaced) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const bool in = i < h && j < w;
  bool changed = false;
  if (in) {
    const int64_t o = (int64_t)i * w + j;
    const double d0 = d[o];
    double res = d0;
    if (c[o] <= alpha) {
      double v[25];
      int n = 0;
      for (int di = -2; di <= 2; ++di) {
        const int qi = i + di;
        if (qi < 0 || qi >= h) continue;
        for (int dj = -2; dj <= 2; ++dj) {
          const int qj = j + dj;
          if (qj < 0 || qj >= w) continue;
          const int64_t q = (int64_t)qi * w + qj;
          if (c[q] > alpha && isfinite(d[q])) v[n++] = d[q];
        }
      }
      if (n > 0) res = lower_median(v, n);
    }
    out[o] = res;
    changed = !(isnan(d0) && isnan(res)) && (res != d0);
  }
  const unsigned bc = __ballot_sync(kFull, changed);
  if ((threadIdx.x & 31) == 0 && bc && replaced)
    atomicAdd(replaced, (unsigned long long)__popc(bc));
}

// ------------------------------------------------------------------ engine
// CostEngine point evaluation (zncc.py:271-287) in fp64, centred.
__device__ double engine_cost(const EngineView& e, int i, int j, int z) {
  const int q = j - e.dir * z;
  if (q < 0 || q > e.W - 1) return -1.0;
  const int64_t pl = (int64_t)i * e.W + j, pr = (int64_t)i * e.W + q;
  const double sl = e.sgL[pl], sr = e.sgR[pr];
  if (!(sl >= e.sigma_eps) || !(sr >= e.sigma_eps)) return -1.0;
  const double ml = e.muL[pl], mr = e.muR[pr];
  const int h2 = e.block / 2;
  double acc = 0.0;
  for (int r = 0; r < e.block; ++r) {
    const int64_t ro = (int64_t)clampi(i + r - h2, 0, e.H - 1) * e.ld;
    for (int c = 0; c < e.block; ++c)
      acc += (e.L[ro + clampi(j + c - h2, 0, e.W - 1)] - ml) *
             (e.R[ro + clampi(q + c - h2, 0, e.W - 1)] - mr);
  }
  const double v = acc / ((double)(e.block * e.block) * sl * sr);
  return fmin(fmax(v, -1.0), 1.0);
}

__global__ void engine_plane_kernel(const EngineView e, int z, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= e.H || j >= e.W) return;
  out[(int64_t)i * e.W + j] = engine_cost(e, i, j, z);
}

__global__ void engine_at_kernel(const EngineView e, const int64_t* rows,
                                 const int64_t* cols, const int64_t* zs,
                                 int64_t n, double* out, int* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = rows[t], j = cols[t], z = zs[t];
  if (z < 0 || z > e.d || i < 0 || i >= e.H || j < 0 || j >= e.W) {
    atomicExch(bad, 1);
    out[t] = -1.0;
    return;
  }
  out[t] = engine_cost(e, (int)i, (int)j, (int)z);
}

__global__ void engine_dsi_kernel(const EngineView e, const int64_t* rows,
                                  const int64_t* cols, int64_t n, double* out,
                                  int* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = n * (int64_t)(e.d + 1);
  if (t >= total) return;
  const int64_t p = t / (e.d + 1);
  const int z = (int)(t - p * (e.d + 1));
  const int64_t i = rows[p], j = cols[p];
  if (i < 0 || i >= e.H || j < 0 || j >= e.W) {
    atomicExch(bad, 1);
    out[t] = -1.0;
    return;
  }
  out[t] = engine_cost(e, (int)i, (int)j, z);
}

__global__ void combine_select_kernel(const int* wc, int h, int w,
                                      const int16_t* fz, const float* fc,
                                      const int16_t* wz, const float* wcst,
                                      double* dout, double* cout) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= h || j >= w) return;
  const int64_t o = (int64_t)i * w + j;
  const bool trusted = wc != nullptr && wc[o] != kWcNone;
  dout[o] = trusted ? (double)wz[o] : (double)fz[o];
  cout[o] = trusted ? (double)wcst[o] : (double)fc[o];
}

__global__ void combine_refine_kernel(const double* din, const double* cin,
                                      int h, int w, double alpha,
                                      const int16_t* nz, const float* nc,
                                      double* dout, double* cout,
                                      unsigned long long* counters) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const bool in = i < h && j < w;
  bool low = false, needed = false;
  if (in) {
    const int64_t o = (int64_t)i * w + j;
    low = cin[o] <= alpha;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        const int qi = i + di, qj = j + dj;
        if (qi >= 0 && qi < h && qj >= 0 && qj < w && cin[(int64_t)qi * w + qj] <= alpha)
          needed = true;
      }
    dout[o] = low ? (double)nz[o] : din[o];
    cout[o] = low ? (double)nc[o] : cin[o];
  }
  const unsigned bl = __ballot_sync(kFull, low);
  const unsigned bn = __ballot_sync(kFull, needed);
  if ((threadIdx.x & 31) == 0) {
    if (bl) atomicAdd(&counters[kCntRefined], (unsigned long long)__popc(bl));
    if (bn) atomicAdd(&counters[kCntNeeded], (unsigned long long)__popc(bn));
  }
}

// ---- shared-memory tiled versions of the per-pixel stage kernels --------
constexpr int kTX = 32, kTY = 8;

// K2, pipeline form: 32 x 32 outputs per CTA (tile reads 1.3x the outputs at
// b = 9 instead of the 8-row tile's 2.5x), sliding box sums in both passes
// (fp64, centred by the tile's first sample as above), input fp64 levels or
// the fp32 level-0 input.
template <int B, typename TIn>
__global__ void __launch_bounds__(256) stats32_kernel(const TIn* img, int h, int w, int64_t ld,
                                                      double sigma_eps, float* mu32, float* is32,
                                                      int64_t lds, int y_base) {
  pdl_wait();
  constexpr int H2 = B / 2, TR = 32 + B - 1, TC = 32 + B - 1;
  constexpr int TCP = TC | 1;   // odd row pitch (doubles): lanes on consecutive rows hit distinct banks
  __shared__ double T[TR][TCP];
  __shared__ double H1[TR][33], H2s[TR][33];
  const int x0 = blockIdx.x * 32, y0 = y_base + blockIdx.y * 32;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const double c = (double)img[(int64_t)clampi(y0, 0, h - 1) * ld + clampi(x0, 0, w - 1)];
#pragma unroll 4
  for (int t = tid; t < TR * TC; t += 256) {
    const int r = t / TC, cc = t - r * TC;
    T[r][cc] = (double)img[(int64_t)clampi(y0 - H2 + r, 0, h - 1) * ld + clampi(x0 - H2 + cc, 0, w - 1)] - c;
  }
  __syncthreads();
  // horizontal: each item = 4 consecutive window sums of one tile row
  // (consecutive lanes on consecutive rows)
  for (int it = tid; it < TR * 8; it += 256) {
    const int r = it % TR, c0 = (it / TR) * 4;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const double v = T[r][c0 + k];
      s1 += v;
      s2 = fma(v, v, s2);
    }
    H1[r][c0] = s1;
    H2s[r][c0] = s2;
#pragma unroll
    for (int e = 1; e < 4; ++e) {
      const double vi = T[r][c0 + e + B - 1], vo = T[r][c0 + e - 1];
      s1 += vi - vo;
      s2 += fma(vi, vi, -vo * vo);
      H1[r][c0 + e] = s1;
      H2s[r][c0 + e] = s2;
    }
  }
  __syncthreads();
  // vertical: thread (x, ty) slides down rows 4 ty .. 4 ty + 3
  const int tx = threadIdx.x, r0 = threadIdx.y * 4;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) s1 += H1[r0 + k][tx], s2 += H2s[r0 + k][tx];
  const int x = x0 + tx;
  constexpr double inv = 1.0 / (double)(B * B);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (e > 0) {
      s1 += H1[r0 + e + B - 1][tx] - H1[r0 + e - 1][tx];
      s2 += H2s[r0 + e + B - 1][tx] - H2s[r0 + e - 1][tx];
    }
    const int y = y0 + r0 + e;
    if (x < w && y < h) {
      const double m1 = s1 * inv, m2 = s2 * inv;
      double var = m2 - m1 * m1;
      if (var <= 1e-9 * m2) {   // flat or near-flat: exact centred recompute
        double ss = 0.0;
        for (int r = 0; r < B; ++r)
#pragma unroll
          for (int cc = 0; cc < B; ++cc) {
            const double dv = T[r0 + e + r][tx + cc] - m1;
            ss = fma(dv, dv, ss);
          }
        var = ss * inv;
      }
      // sigma >= eps <=> var >= eps^2 (no sqrt for the test); 1/sigma
      // through the fp64 reciprocal square root, rounded once to fp32
      mu32[(int64_t)y * lds + x] = (float)(m1 + c);
      is32[(int64_t)y * lds + x] = var >= sigma_eps * sigma_eps ? (float)rsqrt(var) : 0.f;
    }
  }
}

// ---- sweep4 precision guard (kernels.h Sweep4Guard) -----------------------
__device__ __forceinline__ float guard_amp(float mu, float is, float c) {
  return is > 0.f ? fabsf(mu - c) * is + 3.f : 0.f;   // degenerate: cost -1 exactly
}

// per (tile row, column): max aR over the tile row's cost rows y0-1 .. y0+th
__global__ void __launch_bounds__(128) guard_col_kernel(const Sweep4Guard g, int ty0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.w) return;
  const int ty = ty0 + blockIdx.y;
  const int y0 = ty * g.tile_h - kTileOff;
  const float c = *g.cR;
  float m = 0.f;
  for (int y = max(y0 - 1, 0); y <= min(y0 + g.tile_h, g.h - 1); ++y) {
    const int64_t o = (int64_t)y * g.lds + j;
    m = fmaxf(m, guard_amp(g.muR[o], g.isR[o], c));
  }
  g.colR[(int64_t)blockIdx.y * g.w + j] = m;
}

// one warp per tile: max aL over the cost pixels x max aR over their right span
__global__ void __launch_bounds__(32) guard_tile_kernel(const Sweep4Guard g, int ty0) {
  const int tx = blockIdx.x, ty = ty0 + blockIdx.y, lane = threadIdx.x;
  const int x0 = tx * 16, y0 = ty * g.tile_h - kTileOff;
  const int64_t cy = clampi(y0 + g.tile_h / 2, 0, g.h - 1), cx = clampi(x0 + 8, 0, g.w - 1);
  const double cLd = g.L32 ? (double)g.L32[cy * g.ld32 + cx] : g.L[cy * g.ld + cx];
  const float cL = (float)cLd;
  float aL = 0.f, aR = 0.f;
  const int ylo = max(y0 - 1, 0), yhi = min(y0 + g.tile_h, g.h - 1);
  const int xlo = max(x0 - 1, 0), xhi = min(x0 + 16, g.w - 1);
  const int nx = xhi - xlo + 1;
  for (int t = lane; t < (yhi - ylo + 1) * nx; t += 32) {
    const int y = ylo + t / nx, x = xlo + t % nx;
    const int64_t o = (int64_t)y * g.lds + x;
    aL = fmaxf(aL, guard_amp(g.muL[o], g.isL[o], cL));
  }
  const int qlo = max(g.dir > 0 ? x0 - 1 - g.d : x0 - 1, 0);
  const int qhi = min(g.dir > 0 ? x0 + 16 : x0 + 16 + g.d, g.w - 1);
  const float* col = g.colR + (int64_t)blockIdx.y * g.w;
  for (int q = qlo + lane; q <= qhi; q += 32) aR = fmaxf(aR, col[q]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aL = fmaxf(aL, __shfl_xor_sync(kFull, aL, o));
    aR = fmaxf(aR, __shfl_xor_sync(kFull, aR, o));
  }
  if (lane == 0 && aL * aR > kSweep4RiskMax) g.flags[(int64_t)ty * g.flags_ld + tx] = 1u;
}

// prior_eval with the 4x4 spline support of the block staged in smem
constexpr int kPY = 32;   // fine rows per prior_eval block (4 per thread)

__global__ void __launch_bounds__(kTX * kTY) prior_eval_tiled_kernel(
    const int16_t* dco, int64_t ldd, int ch, int cw, const double* coef, int64_t ldc, int h,
    int w, int d, int r, double beta, int* wc, int64_t ldw, unsigned long long* counters,
    RowBand band, double ry, double rx) {
  pdl_wait();
  // 32 fine rows x 32 columns need <= 21 x 21 coefficients (ratio <= 0.52)
  constexpr int CR = 22, CC = 24;
  __shared__ double Cs[CR][CC];
  // spline weights depend only on the row (y) or the column (x): computed
  // once per block row / column; Wx tap-major so lanes read consecutive words
  __shared__ double Wy[kPY][4], Wx[4][kTX];
  __shared__ int Iy[kPY], Ix[kTX];
  const int nh = ch + 2 * kNpad, nw = cw + 2 * kNpad;
  const int i0 = band.lo + blockIdx.y * kPY, j0 = blockIdx.x * kTX;
  const int ylo = (int)floor(((double)i0 + 0.5) * ry - 0.5 + kNpad) - 1;
  const int xlo = (int)floor(((double)j0 + 0.5) * rx - 0.5 + kNpad) - 1;
  const int tid = threadIdx.y * kTX + threadIdx.x;
  {
    constexpr int kPer = (CR * CC + kTX * kTY - 1) / (kTX * kTY);
    double v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + kTX * kTY * k;
      const int a = t / CC, b = t - a * CC;
      v[k] = t < CR * CC ? coef[(int64_t)clampi(ylo + a, 0, nh - 1) * ldc +
                                clampi(xlo + b, 0, nw - 1)]
                         : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + kTX * kTY * k;
      if (t < CR * CC) Cs[t / CC][t % CC] = v[k];
    }
  }
  if (tid < kTX) {
    const double x = ((double)(j0 + tid) + 0.5) * rx - 0.5 + kNpad;
    const double fx = floor(x);
    double wt[4];
    bspline_w(x - fx, wt);
#pragma unroll
    for (int b = 0; b < 4; ++b) Wx[b][tid] = wt[b];
    Ix[tid] = (int)fx - 1 - xlo;
  } else if (tid < kTX + kPY) {
    const int rr = tid - kTX;
    const double y = ((double)(i0 + rr) + 0.5) * ry - 0.5 + kNpad;
    const double fy = floor(y);
    bspline_w(y - fy, Wy[rr]);
    Iy[rr] = (int)fy - 1 - ylo;
  }
  __syncthreads();
  const int j = j0 + threadIdx.x;
  double wx[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) wx[b] = Wx[b][threadIdx.x];
  const int ix = Ix[threadIdx.x];
  unsigned ntr = 0;
  unsigned long long wsum = 0, wmax = 0;
#pragma unroll
  for (int q = 0; q < kPY / kTY; ++q) {
    const int ty = threadIdx.y + kTY * q;
    const int i = i0 + ty;
    if (i < band.hi && i < h && j < w) {
      const double* wy = Wy[ty];
      const int iy = Iy[ty];   // within the tile
      double chat = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double rr = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) rr += wx[b] * Cs[iy + a][ix + b];
        chat += wy[a] * rr;
      }
      chat = fmin(fmax(chat, -1.0), 1.0);
      const int center = 2 * (int)dco[(int64_t)(i >> 1) * ldd + (j >> 1)];
      const bool ok = (center + r >= 0) && (center - r <= d);
      const bool trusted = (chat > beta) && ok;
      wc[(int64_t)i * ldw + j] = trusted ? center : kWcNone;
      if (trusted && i >= band.cnt_lo && i < band.cnt_hi) {
        const unsigned long long ws =
            (unsigned long long)(min(center + r, d) - max(center - r, 0) + 1);
        ntr += 1;
        wsum += ws;
        wmax = ws > wmax ? ws : wmax;
      }
    }
  }
  const int slot[3] = {kCntTrusted, kCntTrustedEvals, kCntWindowMax};
  const unsigned long long val[3] = {ntr, wsum, wmax};
  const bool mx[3] = {false, false, true};
  block_accumulate<3>(counters, slot, val, mx);
}

// Sorting network for 24 keys: Batcher's odd-even merge sort for 32 inputs
// with the comparators that touch inputs 24..31 removed (those would hold
// +inf sentinels and never move).  Generated and checked (random inputs,
// 0/1 principle) by tools/median_net.py.
constexpr int kMedNetLen = 132;
__device__ constexpr unsigned char kMedNet[2 * kMedNetLen] = {0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,18,19,20,21,22,23,0,2,1,3,4,6,5,7,8,10,9,11,12,14,13,15,16,18,17,19,20,22,21,23,1,2,5,6,9,10,13,14,17,18,21,22,0,4,1,5,2,6,3,7,8,12,9,13,10,14,11,15,16,20,17,21,18,22,19,23,2,4,3,5,10,12,11,13,18,20,19,21,1,2,3,4,5,6,9,10,11,12,13,14,17,18,19,20,21,22,0,8,1,9,2,10,3,11,4,12,5,13,6,14,7,15,4,8,5,9,6,10,7,11,2,4,3,5,6,8,7,9,10,12,11,13,18,20,19,21,1,2,3,4,5,6,7,8,9,10,11,12,13,14,17,18,19,20,21,22,0,16,1,17,2,18,3,19,4,20,5,21,6,22,7,23,8,16,9,17,10,18,11,19,12,20,13,21,14,22,15,23,4,8,5,9,6,10,7,11,12,16,13,17,14,18,15,19,2,4,3,5,6,8,7,9,10,12,11,13,14,16,15,17,18,20,19,21,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,18,19,20,21,22};

// selective median (pipeline) with the 5x5 neighbourhood staged in smem
constexpr int kMY = 32;   // rows per median block (4 per thread)

__device__ __forceinline__ unsigned min_s16x2(unsigned a, unsigned b) {
  unsigned r;
  asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned max_s16x2(unsigned a, unsigned b) {
  unsigned r;
  asm("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// selective_median (matcher.py:323-359) on a 32 x kMY tile (+2 halo): the
// alpha gate is applied once per tile element (Qs = disparity where C > alpha,
// else the +inf sentinel 0x7FFF, int16), low pixels (C <= alpha) go to a
// block-local work list, and each thread sorts the 24 neighbour slots of TWO
// listed pixels at once: one pixel per 16-bit half, the 132-comparator
// network (kMedNet) as packed VIMNMX.S16x2, then the lower median (n-1)/2 of
// each half's n qualifying values.
__global__ void __launch_bounds__(kTX * kTY) median_tiled_kernel(
    const int16_t* d, const float* c, const uint8_t* low, int64_t ld, int h, int w,
    double alpha, int16_t* out, unsigned long long* counters, RowBand band) {
  pdl_wait();
  constexpr int TR = kMY + 4, TC = kTX + 4;
  constexpr short kInf = 0x7FFF;
  __shared__ short Qs[TR][TC];
  __shared__ short Ds[TR][TC];
  __shared__ uint8_t Lw[TR][TC];
  const int x0 = blockIdx.x * kTX, y0 = band.lo + blockIdx.y * kMY;
  const int tid = threadIdx.y * kTX + threadIdx.x;
  {
    // all of a thread's loads in flight before the stores
    constexpr int kPer = (TR * TC + kTX * kTY - 1) / (kTX * kTY);
    float cv[kPer];
    int16_t dv[kPer];
    uint8_t lv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + kTX * kTY * k;
      const int a = t / TC, b = t - a * TC;
      const int gy = y0 - 2 + a, gx = x0 - 2 + b;
      cv[k] = -2.f;     // below any legal alpha: never qualifies (matcher.py:345)
      dv[k] = 0;
      lv[k] = 0;
      if (t < TR * TC && gy >= 0 && gy < h && gx >= 0 && gx < w) {
        const int64_t o = (int64_t)gy * ld + gx;
        cv[k] = c[o];
        dv[k] = d[o];
        lv[k] = low[o];
      }
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = tid + kTX * kTY * k;
      if (t < TR * TC) {
        const int a = t / TC, b = t - a * TC;
        Qs[a][b] = (double)cv[k] > alpha ? dv[k] : kInf;
        Ds[a][b] = dv[k];
        Lw[a][b] = lv[k] | ((double)cv[k] <= alpha ? 2 : 0);   // bit 1: C <= alpha
      }
    }
  }
  __shared__ short list[kMY * kTX];
  __shared__ int nlist;
  if (tid == 0) nlist = 0;
  __syncthreads();
  const int j = x0 + threadIdx.x;
  unsigned nneeded = 0;
#pragma unroll
  for (int q = 0; q < kMY / kTY; ++q) {
    const int py = threadIdx.y + kTY * q;
    const int i = y0 + py;
    if (i < band.hi && i < h && j < w) {
      const int ty = py + 2, tx = threadIdx.x + 2;
      bool needed = false;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) needed |= (Lw[ty + di][tx + dj] & 1) != 0;
      nneeded += (needed && i >= band.cnt_lo && i < band.cnt_hi) ? 1u : 0u;
      // low-confidence pixels go to the work list; the others keep their
      // disparity
      if (!(Lw[ty][tx] & 2)) out[(int64_t)i * ld + j] = Ds[ty][tx];
    }
    // the list keeps each warp's row in order (one atomic per warp), so the
    // pixel pairs sorted together are neighbours with overlapping windows
    const bool lw = i < band.hi && i < h && j < w && (Lw[py + 2][threadIdx.x + 2] & 2);
    const unsigned m = __ballot_sync(0xffffffffu, lw);
    int base = 0;
    if (threadIdx.x == 0 && m) base = atomicAdd(&nlist, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lw) list[base + __popc(m & ((1u << threadIdx.x) - 1u))] = (short)(py * kTX + threadIdx.x);
  }
  __syncthreads();
  unsigned nchanged = 0;
  const int n_items = nlist;
  for (int k = 2 * tid; k < n_items; k += 2 * kTX * kTY) {
    const bool two = k + 1 < n_items;
    const int pa = list[k], pb = two ? list[k + 1] : pa;
    const int tya = pa / kTX + 2, txa = pa % kTX + 2;
    const int tyb = pb / kTX + 2, txb = pb % kTX + 2;
    unsigned v[24];
    int na = 0, nb = 0;
#pragma unroll
    for (int t = 0; t < 24; ++t) {
      const int u = t < 12 ? t : t + 1;          // skip the centre (slot 12)
      const int di = u / 5 - 2, dj = u % 5 - 2;
      const short qa = Qs[tya + di][txa + dj], qb = Qs[tyb + di][txb + dj];
      na += qa != kInf;
      nb += qb != kInf;
      v[t] = (unsigned)(unsigned short)qa | ((unsigned)(unsigned short)qb << 16);
    }
#pragma unroll
    for (int cc = 0; cc < kMedNetLen; ++cc) {
      const int i0 = kMedNet[2 * cc], i1 = kMedNet[2 * cc + 1];
      const unsigned x = v[i0], y = v[i1];
      v[i0] = min_s16x2(x, y);
      v[i1] = max_s16x2(x, y);
    }
    const int ma = (na - 1) >> 1, mb = (nb - 1) >> 1;
    unsigned sa = v[0], sb = v[0];
#pragma unroll
    for (int t = 1; t < 24; ++t) {
      sa = (ma == t) ? v[t] : sa;
      sb = (mb == t) ? v[t] : sb;
    }
    {
      const int16_t d0 = Ds[tya][txa];
      const int16_t res = na > 0 ? (int16_t)(sa & 0xffffu) : d0;
      const int gi = y0 + tya - 2, gj = x0 + txa - 2;
      out[(int64_t)gi * ld + gj] = res;
      nchanged += (res != d0 && gi >= band.cnt_lo && gi < band.cnt_hi) ? 1u : 0u;
    }
    if (two) {
      const int16_t d0 = Ds[tyb][txb];
      const int16_t res = nb > 0 ? (int16_t)(sb >> 16) : d0;
      const int gi = y0 + tyb - 2, gj = x0 + txb - 2;
      out[(int64_t)gi * ld + gj] = res;
      nchanged += (res != d0 && gi >= band.cnt_lo && gi < band.cnt_hi) ? 1u : 0u;
    }
  }
  const int slot[2] = {kCntMedianReplaced, kCntNeeded};
  const unsigned long long val[2] = {nchanged, nneeded};
  const bool mx[2] = {false, false};
  block_accumulate<2>(counters, slot, val, mx);
}

// ------------------------------------------------------------------ staging
template <typename TIn>
__global__ void __launch_bounds__(256) prep_staging_kernel(const TIn* R, int64_t ld,
                                                           const float* muR, const float* isR,
                                                           int64_t lds, int h, int w, int pc,
                                                           float* Rp, float2* Mp, int64_t ldp,
                                                           int y0, int y1, const float* cR) {
  pdl_wait();
  // 4 consecutive padded columns per thread (ldp and pc are multiples of 4:
  // one float4 and two float4 stores)
  const int xp0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int y = y0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (y >= h || y >= y1 || xp0 >= w + 2 * pc) return;
  // the level's right offset: the pipeline's constant (valid in any row
  // band), else (stage API, whole level) the box mean at the image centre
  const float c = cR ? *cR : muR[(int64_t)(h / 2) * lds + w / 2];
  const float qnan = __int_as_float(0x7fc00000);
  float r4[4];
  float2 m4[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int x = xp0 + e - pc;
    const int xc = clampi(x, 0, w - 1);
    // fl32(R - c): for the fp32 level-0 input the fp32 subtraction is that rounding
    r4[e] = (float)((double)R[(int64_t)y * ld + xc] - (double)c);
    m4[e] = make_float2(0.f, qnan);
    if (x >= 0 && x < w) {
      const float is = isR[(int64_t)y * lds + x];
      // 0.5/sigma_R: the sweep computes the half-range cost c/2 + 1/2
      m4[e] = make_float2(muR[(int64_t)y * lds + x] - c, is > 0.f ? 0.5f * is : qnan);
    }
  }
  const int64_t o = (int64_t)y * ldp + xp0;
  *reinterpret_cast<float4*>(Rp + o) = make_float4(r4[0], r4[1], r4[2], r4[3]);
  reinterpret_cast<float4*>(Mp + o)[0] = make_float4(m4[0].x, m4[0].y, m4[1].x, m4[1].y);
  reinterpret_cast<float4*>(Mp + o)[1] = make_float4(m4[2].x, m4[2].y, m4[3].x, m4[3].y);
}

// ------------------------------------------------------------------ evaluate
// evaluation.py:77-109: on pixels valid in both maps, |d*scale - gt| vs the
// bad thresholds, mean absolute error; invalid counts.  counts[] = {evaluated,
// bad_t0, bad_t1, bad_t2, gt_invalid, output_invalid}.
__global__ void evaluate_kernel(const double* d, const double* gt, const uint8_t* gt_invalid,
                                int64_t n, double scale, double t0, double t1, double t2,
                                unsigned long long* counts, double* abs_sum) {
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[k];
    const bool out_bad = !isfinite(v);
    const bool gt_bad = gt_invalid[k] != 0;
    c[4] += gt_bad;
    c[5] += out_bad;
    if (!out_bad && !gt_bad) {
      const double e = fabs(v * scale - gt[k]);
      c[0] += 1;
      c[1] += e > t0;
      c[2] += e > t1;
      c[3] += e > t2;
      acc += e;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 6; ++q) c[q] += __shfl_xor_sync(kFull, c[q], o);
    acc += __shfl_xor_sync(kFull, acc, o);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q)
      if (c[q]) atomicAdd(&counts[q], c[q]);
    atomicAdd(abs_sum, acc);
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_f32_to_f64(const float* a, const float* b, int h, int w,
                              int64_t ld_in, double* oa, double* ob,
                              int64_t ld_out, cudaStream_t s) {
  dim3 blk(64, 4);
  f32_to_f64_kernel<<<grid2d(w, h, blk, b ? 2 : 1), blk, 0, s>>>(a, b, h, w, ld_in, oa, ob, ld_out);
  return cudaGetLastError();
}

cudaError_t launch_evaluate(const double* d, const double* gt, const uint8_t* gt_invalid,
                            int64_t n, double scale, const double* taus,
                            unsigned long long* counts, double* abs_sum, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  evaluate_kernel<<<blocks, 256, 0, s>>>(d, gt, gt_invalid, n, scale, taus[0], taus[1], taus[2],
                                         counts, abs_sum);
  return cudaGetLastError();
}

template <typename TIn>
cudaError_t launch_prep_staging_t(const TIn* R, int64_t ld, const float* muR, const float* isR,
                                  int64_t lds, int h, int w, int pc, float* Rp, float2* Mp,
                                  int64_t ldp, cudaStream_t s, int y0, int y1, const float* cR) {
  if (y1 < 0 || y1 > h) y1 = h;
  if (y1 <= y0) return cudaSuccess;
  dim3 blk(64, 4);
  return launch_pdl(prep_staging_kernel<TIn>, grid2d((w + 2 * pc + 3) / 4, y1 - y0, blk), blk, 0,
                    s, R, ld, muR, isR, lds, h, w, pc, Rp, Mp, ldp, y0, y1, cR);
}
cudaError_t launch_prep_staging(const double* R, int64_t ld, const float* muR, const float* isR,
                                int64_t lds, int h, int w, int pc, float* Rp, float2* Mp,
                                int64_t ldp, cudaStream_t s, int y0, int y1, const float* cR) {
  return launch_prep_staging_t(R, ld, muR, isR, lds, h, w, pc, Rp, Mp, ldp, s, y0, y1, cR);
}
cudaError_t launch_prep_staging(const float* R, int64_t ld, const float* muR, const float* isR,
                                int64_t lds, int h, int w, int pc, float* Rp, float2* Mp,
                                int64_t ldp, cudaStream_t s, int y0, int y1, const float* cR) {
  return launch_prep_staging_t(R, ld, muR, isR, lds, h, w, pc, Rp, Mp, ldp, s, y0, y1, cR);
}

// The pipeline's right-image offset c (every level): the level-0 right
// sample at the image centre, so any row band sees the same constant.
__global__ void centre_sample_kernel(const float* in32, const double* in64, int64_t ld, int h,
                                     int w, float* out) {
  pdl_wait();
  const int64_t o = (int64_t)(h / 2) * ld + w / 2;
  *out = in32 ? in32[o] : (float)in64[o];
}

cudaError_t launch_centre_sample(const float* in32, const double* in64, int64_t ld, int h,
                                 int w, float* out, cudaStream_t s) {
  centre_sample_kernel<<<1, 1, 0, s>>>(in32, in64, ld, h, w, out);
  return cudaGetLastError();
}

cudaError_t launch_downsample(const double* in0, const double* in1, int h,
                              int w, int64_t ld_in, double* out0, double* out1,
                              int64_t ld_out, cudaStream_t s, int i0, int i1) {
  const int oh = (h + 1) / 2, ow = (w + 1) / 2;
  if (i1 < 0 || i1 > oh) i1 = oh;
  if (i1 <= i0) return cudaSuccess;
  const dim3 g((ow + 31) / 32, (i1 - i0 + 15) / 16, in1 ? 2 : 1);
  return launch_pdl(downsample_tile_kernel<double>, g, dim3(256), 0, s, in0, in1, h, w, ld_in,
                    out0, out1, ld_out, oh, ow, i0, i1);
}

// binomial_smooth (pyramid.py:65-68): the same separable 5-tap filter at
// full resolution (step 1, no decimation); stage API only
cudaError_t launch_binomial_smooth(const double* in, int h, int w, int64_t ld_in, double* out,
                                   int64_t ld_out, cudaStream_t s) {
  dim3 blk(32, 8);
  return launch_pdl(downsample_kernel<double, false>, grid2d(w, h, blk, 1), blk, 0, s, in,
                    (const double*)nullptr, h, w, ld_in, out, (double*)nullptr, ld_out, h, w,
                    (double*)nullptr, (double*)nullptr, (int64_t)0, 0, h, 1);
}

cudaError_t launch_downsample_f32(const float* in0, const float* in1, int h, int w,
                                  int64_t ld_in, double* out0, double* out1, int64_t ld_out,
                                  double* copy0, double* copy1, int64_t ld_copy,
                                  cudaStream_t s, int i0, int i1) {
  const int oh = (h + 1) / 2, ow = (w + 1) / 2;
  if (i1 < 0 || i1 > oh) i1 = oh;
  if (i1 <= i0) return cudaSuccess;
  dim3 blk(32, 8);
  if (copy0 == nullptr)   // level 0 stays fp32 (its consumers read the input)
    return launch_pdl(downsample_tile_kernel<float>, dim3((ow + 31) / 32, (i1 - i0 + 15) / 16, 2),
                      dim3(256), 0, s, in0, in1, h, w, ld_in, out0, out1, ld_out, oh, ow, i0, i1);
  return launch_pdl(downsample_kernel<float, true>, grid2d(ow, i1 - i0, blk, 2), blk, 0, s, in0,
                    in1, h, w, ld_in, out0, out1, ld_out, oh, ow, copy0, copy1, ld_copy, i0, i1, 2);
}

template <typename TIn>
cudaError_t launch_stats32(const TIn* img, int h, int w, int64_t ld, int b, double sigma_eps,
                           float* mu, float* is, int64_t lds, cudaStream_t s, int y0, int y1) {
  const int yb = (y0 / 32) * 32;   // whole-image tile grid
  const dim3 blk(32, 8), gr((w + 31) / 32, (y1 - yb + 31) / 32);
  auto go = [&](auto kern) {
    return launch_pdl(kern, gr, blk, 0, s, img, h, w, ld, sigma_eps, mu, is, lds, yb);
  };
  switch (b) {
    case 3: return go(stats32_kernel<3, TIn>);
    case 5: return go(stats32_kernel<5, TIn>);
    case 7: return go(stats32_kernel<7, TIn>);
    case 9: return go(stats32_kernel<9, TIn>);
    case 11: return go(stats32_kernel<11, TIn>);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_stats_f32(const float* img, int h, int w, int64_t ld, int b, double sigma_eps,
                             float* mu, float* is, int64_t lds, cudaStream_t s, int y0, int y1) {
  if (y1 < 0 || y1 > h) y1 = h;
  if (y1 <= y0) return cudaSuccess;
  if (b <= 11) return launch_stats32(img, h, w, ld, b, sigma_eps, mu, is, lds, s, y0, y1);
  return cudaErrorInvalidValue;   // fp32 input: level 0 of sweep4 levels (b <= 11)
}

cudaError_t launch_stats_f32(const double* img, int h, int w, int64_t ld,
                             int b, double sigma_eps, float* mu, float* is,
                             int64_t lds, cudaStream_t s, int y0, int y1) {
  if (y1 < 0 || y1 > h) y1 = h;
  if (y1 <= y0) return cudaSuccess;
  if (b <= 11) return launch_stats32(img, h, w, ld, b, sigma_eps, mu, is, lds, s, y0, y1);
  dim3 blk(32, 8);
  const int yb = (y0 / kTY) * kTY;   // whole-image tile grid
  const dim3 gr = grid2d(w, y1 - yb, blk);
  stats_kernel<false><<<gr, blk, 0, s>>>(img, h, w, ld, b, sigma_eps, mu, is, nullptr, nullptr,
                                          lds, yb);
  return cudaGetLastError();
}

cudaError_t launch_stats_f64(const double* img, int h, int w, int64_t ld,
                             int b, double* mu, double* sigma, cudaStream_t s) {
  dim3 blk(32, 8);
  stats_kernel<true><<<grid2d(w, h, blk), blk, 0, s>>>(img, h, w, ld, b, 0.0, nullptr,
                                                        nullptr, mu, sigma, 0);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fir(const T* cin, int ch, int cw, int64_t ldcin, double* coef, int64_t ldc,
                       cudaStream_t s, int r0, int r1) {
  const int nh = ch + 2 * kNpad, nw = cw + 2 * kNpad;
  constexpr size_t smem = (sizeof(T) * kFE * (kFE + 1) + 7) / 8 * 8 +
                          sizeof(double) * kFT * (kFE + 1);
  static SmemAttr attr;
  if (cudaError_t e = attr.ensure(bspline_fir_kernel<T>, smem); e != cudaSuccess) return e;
  // coefficient rows [r0, r1) of the padded grid (r1 < 0: all), whole tiles
  if (r1 < 0 || r1 > nh) r1 = nh;
  r0 = std::max(r0, 0);
  if (r1 <= r0) return cudaSuccess;
  const int t0 = r0 / kFT, t1 = (r1 + kFT - 1) / kFT;
  const dim3 grid((nw + kFT - 1) / kFT, t1 - t0);
  bspline_fir_kernel<T><<<grid, 256, smem, s>>>(cin, ch, cw, ldcin, coef, ldc, t0);
  return cudaGetLastError();
}

cudaError_t launch_bspline_prefilter(const float* c32, const double* c64,
                                     int ch, int cw, int64_t ldcin,
                                     double* coef, int64_t ldc, cudaStream_t s, int r0, int r1) {
  return c32 ? launch_fir(c32, ch, cw, ldcin, coef, ldc, s, r0, r1)
             : launch_fir(c64, ch, cw, ldcin, coef, ldc, s, r0, r1);
}

void prior_coef_rows(int ch, int h, RowBand rows, int* r0, int* r1) {
  const double ry = (double)ch / (double)h;
  const int lo = std::max(rows.lo, 0), hi = std::max(rows.hi, lo + 1);
  *r0 = (int)floor(((double)lo + 0.5) * ry - 0.5 + kNpad) - 1 - 2;
  *r1 = (int)floor(((double)(hi - 1) + 0.5) * ry - 0.5 + kNpad) + 3 + 2;
}

cudaError_t launch_prior_eval(const int16_t* dcoarse, int64_t ldd, int ch,
                              int cw, const double* coef, int64_t ldc, int h,
                              int w, int d, int radius, double beta, int* wc,
                              int64_t ldw, unsigned long long* counters,
                              RowBand rows, cudaStream_t s) {
  dim3 blk(32, 8);
  const dim3 g((w + 31) / 32, (rows.hi - rows.lo + kPY - 1) / kPY);
  return launch_pdl(prior_eval_tiled_kernel, g, blk, 0, s, dcoarse, ldd, ch, cw, coef, ldc, h, w,
                    d, radius, beta, wc, ldw, counters, rows, (double)ch / (double)h,
                    (double)cw / (double)w);
}

cudaError_t launch_prior_maps(const double* d_hat, const double* c_hat, int h,
                              int w, int d, int radius, double beta, int* wc,
                              int64_t ldw, unsigned long long* counters,
                              cudaStream_t s) {
  dim3 blk(32, 8);
  prior_maps_kernel<<<grid2d(w, h, blk), blk, 0, s>>>(d_hat, c_hat, h, w, d, radius, beta,
                                                       wc, ldw, counters);
  return cudaGetLastError();
}

cudaError_t launch_upsample(const double* dcoarse, int ch, int cw,
                            const double* coef, int64_t ldc, int h, int w,
                            double* d_hat, double* c_hat, cudaStream_t s) {
  dim3 blk(32, 8);
  upsample_kernel<<<grid2d(w, h, blk), blk, 0, s>>>(dcoarse, ch, cw, coef, ldc, h, w, d_hat,
                                                     c_hat);
  return cudaGetLastError();
}

cudaError_t launch_median_pipeline(const int16_t* d, const float* c,
                                   const uint8_t* low, int64_t ld, int h,
                                   int w, double alpha, int16_t* out,
                                   unsigned long long* counters, RowBand rows,
                                   cudaStream_t s) {
  dim3 blk(32, 8);
  const dim3 g((w + 31) / 32, (rows.hi - rows.lo + kMY - 1) / kMY);
  cudaError_t e = launch_pdl(median_tiled_kernel, g, blk, 0, s, d, c, low, ld, h, w, alpha, out,
                             counters, rows);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_median_f64(const double* d, const double* c, int h, int w,
                              double alpha, double* out,
                              unsigned long long* replaced, cudaStream_t s) {
  dim3 blk(32, 8);
  median_f64_kernel<<<grid2d(w, h, blk), blk, 0, s>>>(d, c, h, w, alpha, out, replaced);
  return cudaGetLastError();
}

cudaError_t launch_engine_plane(const EngineView& e, int z, double* out,
                                cudaStream_t s) {
  dim3 blk(32, 8);
  engine_plane_kernel<<<grid2d(e.W, e.H, blk), blk, 0, s>>>(e, z, out);
  return cudaGetLastError();
}

cudaError_t launch_engine_at(const EngineView& e, const int64_t* rows,
                             const int64_t* cols, const int64_t* z, int64_t n,
                             double* out, int* bad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  engine_at_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(e, rows, cols, z, n, out, bad);
  return cudaGetLastError();
}

cudaError_t launch_engine_dsi(const EngineView& e, const int64_t* rows,
                              const int64_t* cols, int64_t n, double* out,
                              int* bad, cudaStream_t s) {
  const int64_t total = n * (int64_t)(e.d + 1);
  if (total <= 0) return cudaSuccess;
  engine_dsi_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(e, rows, cols, n, out, bad);
  return cudaGetLastError();
}

cudaError_t launch_combine_select(const int* wc, int h, int w,
                                  const int16_t* fz, const float* fc,
                                  const int16_t* wz, const float* wcst,
                                  double* dout, double* cout, cudaStream_t s) {
  dim3 blk(32, 8);
  combine_select_kernel<<<grid2d(w, h, blk), blk, 0, s>>>(wc, h, w, fz, fc, wz, wcst, dout,
                                                           cout);
  return cudaGetLastError();
}

cudaError_t launch_combine_refine(const double* din, const double* cin, int h,
                                  int w, double alpha, const int16_t* nz,
                                  const float* nc, double* dout, double* cout,
                                  unsigned long long* counters, cudaStream_t s) {
  dim3 blk(32, 8);
  combine_refine_kernel<<<grid2d(w, h, blk), blk, 0, s>>>(din, cin, h, w, alpha, nz, nc, dout,
                                                           cout, counters);
  return cudaGetLastError();
}

cudaError_t launch_sweep4_guard(const Sweep4Guard& g, RowBand rows, cudaStream_t s) {
  if (g.flags == nullptr || rows.hi <= rows.lo) return cudaSuccess;
  const int ty0 = tile_row(rows.lo, g.tile_h), ty1 = tile_row(rows.hi - 1, g.tile_h);
  const int nty = ty1 - ty0 + 1;
  guard_col_kernel<<<dim3((g.w + 127) / 128, nty), 128, 0, s>>>(g, ty0);
  guard_tile_kernel<<<dim3((g.w + 15) / 16, nty), 32, 0, s>>>(g, ty0);
  return cudaGetLastError();
}

}  // namespace mshbm
