// Dense fused ZNCC z-sweep (one launch per pyramid level).
//
// Replaces, for one level, the reference's
//   match_coarsest / CostEngine.plane+full_volume (matcher.py:184-193,
//   zncc.py:202-249), select_with_prior's window and full-range branches
//   (matcher.py:263-320, CostEngine.at / dsi_rows zncc.py:251-302) and
//   refine_level's 3x3-summed re-selection (matcher.py:196-233),
// without ever materialising the disparity-space image.
//
// Layout: a CTA is NR warps x 32 lanes; lane l / warp w own pixel
// (y0-1+w, x0-1+l).  Border lanes/warps are the 1-pixel halo the 3x3 cost
// sums need; inner outputs are 30 x (NR-2) per CTA.  Each thread keeps its
// own left window centred in fp64 and rounded once to fp32 (L~ = L - muL),
// and sweeps z in chunks of ZC: the right-image strip of the chunk
// (rows of the window, columns of all 32 lanes x ZC shifts) is staged in
// shared memory offset by a per-CTA constant cR, and the per-thread
// cross sums S[zz] = sum L~ (R - cR) are register-blocked over the chunk
// (ZC+B-1 shared loads feed ZC*B FMAs per window row).  The bias term
// (muR(q) - cR) * sum(L~) restores the exact centred covariance.
// Per z the cost feeds three strict-'>' winner-take-all states held in
// registers (full range, +-r prior window, 3x3 sum); horizontal
// neighbours of the 3x3 sum come from warp shuffles, vertical ones from a
// shared-memory row exchange.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace mshbm {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// One chunk of NZ disparities starting at z0, reading the staged strip of a
// ZC-wide chunk (NZ <= ZC; the tail of the range uses NZ = 4 with masking).
template <int B, int DIR, int ZC, int NR, int NZ>
__device__ __forceinline__ void sweep_chunk(
    const float (&Rs)[NR + B - 1][30 + B + ZC], const float2 (&Ms)[NR][31 + ZC],
    float (&Hs)[ZC][NR][32], const float (&Lt)[B][B], float sumLt, int z0, int zoff,
    int zend, bool inimg, int lane, int wp, float& bF, int& zF, bool wchunk, int wlo,
    int whi, float& bW, int& zW) {
  float S[NZ];
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) S[zz] = 0.f;
  // window rows x staged columns; (c, zz) pairs sharing a column reuse one load
#pragma unroll
  for (int r = 0; r < B; ++r) {
    const float* rp = &Rs[wp + r][lane];
#pragma unroll
    for (int e = 0; e < NZ + B - 1; ++e) {
      // strip index relative to the chunk: DIR>0 -> g = ZC-1-(zoff+zz)
      const int eo = DIR > 0 ? (ZC - NZ - zoff) + e : zoff + e;
      const float v = rp[eo];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const int g = e - c;
        if (g >= 0 && g < NZ) {
          const int zz = DIR > 0 ? (NZ - 1 - g) : g;
          S[zz] = fmaf(Lt[r][c], v, S[zz]);
        }
      }
    }
  }
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) {
    const int z = z0 + zoff + zz;
    const int g = DIR > 0 ? (ZC - 1 - (zoff + zz)) : (zoff + zz);
    const float2 mi = Ms[wp][lane + g];          // (muR - cR, 1/sigma_R); NaN = invalid
    float rho = fmaf(-mi.x, sumLt, S[zz]) * mi.y;  // NaN for invalid q / flat left block
    rho = fminf(fmaxf(rho, -1.f), 1.f);            // fmaxf(NaN, -1) = -1
    if (NZ < ZC && z > zend) rho = -3.f;           // masked tail slot
    if (rho > bF) { bF = rho; zF = z; }
    if (wchunk) {   // warp-uniform: some lane's prior window meets this chunk
      if (z >= wlo && z <= whi && rho > bW) { bW = rho; zW = z; }
    }
    const float o = inimg ? rho : 0.f;
    const float hl = __shfl_up_sync(kFull, o, 1);
    const float hr = __shfl_down_sync(kFull, o, 1);
    Hs[zoff + zz][wp][lane] = (hl + o) + hr;
  }
}

template <int B, int DIR, int ZC, int NR, int MINB>
__global__ void __launch_bounds__(NR * 32, MINB)
sweep_kernel(const SweepArgs a) {
  constexpr int H2 = B / 2;
  constexpr int NT = NR * 32;
  constexpr int RW = 30 + B + ZC;  // 32 + (B-1) + (ZC-1) staged columns
  constexpr int RR = NR + B - 1;   // staged rows
  constexpr int SW = 31 + ZC;      // 32 + (ZC-1) stats columns
  constexpr int KR = (RR * RW + NT - 1) / NT;   // staged R values per thread
  constexpr int KS = (NR * SW + NT - 1) / NT;   // staged stats per thread
  using RsT = float[RR][RW];
  using MsT = float2[NR][SW];
  using HsT = float[ZC][NR][32];
  extern __shared__ float4 smem4[];
  RsT* Rs = reinterpret_cast<RsT*>(smem4);                 // [2]
  MsT* Ms = reinterpret_cast<MsT*>(Rs + 2);                // [2]
  HsT* Hs = reinterpret_cast<HsT*>(Ms + 2);                // [2]

  const int lane = threadIdx.x & 31;
  const int wp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 30;
  const int y0 = a.rows.lo + blockIdx.y * (NR - 2);
  const int i = y0 - 1 + wp;
  const int j = x0 - 1 + lane;
  const int H = a.H, W = a.W, d = a.d;
  const bool inimg = (i >= 0) && (i < H) && (j >= 0) && (j < W);
  const bool inner = inimg && lane >= 1 && lane <= 30 && wp >= 1 && wp <= NR - 2;
  const float qnan = __int_as_float(0x7fc00000);

  // per-CTA constant offset of the right image (tile-centre sample)
  const double cR = a.Rv(clampi(y0 + NR / 2 - 1, 0, H - 1), clampi(x0 + 15, 0, W - 1));
  const float cRf = (float)cR;

  // ---- staging: global -> registers (prefetch) -> shared (double buffer)
  double pr[KR];
  float2 pm[KS];
  auto fetch = [&](int z0) {
    const int s0 = DIR > 0 ? (x0 - 1 - H2 - z0 - (ZC - 1)) : (x0 - 1 - H2 + z0);
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < RR * RW) {
        const int rr = t / RW, e = t - rr * RW;
        const int gi = clampi(y0 - 1 - H2 + rr, 0, H - 1);
        const int gc = clampi(s0 + e, 0, W - 1);
        pr[k] = a.Rv(gi, gc);
      }
    }
    const int q0 = DIR > 0 ? (x0 - 1 - z0 - (ZC - 1)) : (x0 - 1 + z0);
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < NR * SW) {
        const int rr = t / SW, e = t - rr * SW;
        const int gi = clampi(y0 - 1 + rr, 0, H - 1);
        const int gq = q0 + e;
        if (gq >= 0 && gq < W) {
          const int64_t o = (int64_t)gi * a.lds + gq;
          const float is = a.isR[o];
          pm[k] = make_float2(is > 0.f ? a.muR[o] - cRf : qnan, is);
        } else {
          pm[k] = make_float2(qnan, 0.f);   // right centre outside the image
        }
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < RR * RW) {
        const int rr = t / RW, e = t - rr * RW;
        Rs[buf][rr][e] = (float)(pr[k] - cR);
      }
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < NR * SW) {
        const int rr = t / SW, e = t - rr * SW;
        Ms[buf][rr][e] = pm[k];
      }
    }
  };
  fetch(0);

  // ---- left tile (fp64) through shared memory, aliasing the Hs buffers
  // (first written after the barrier that follows store(0))
  constexpr int LC = 31 + B;
  using LtT = double[RR][LC];
  static_assert(sizeof(LtT) <= 2 * sizeof(HsT), "left tile must fit in Hs");
  LtT& Ls = *reinterpret_cast<LtT*>(Hs);
  for (int t = threadIdx.x; t < RR * LC; t += NT) {
    const int rr = t / LC, e = t - rr * LC;
    Ls[rr][e] = a.Lv(clampi(y0 - 1 - H2 + rr, 0, H - 1), clampi(x0 - 1 - H2 + e, 0, W - 1));
  }
  __syncthreads();

  // ---- left window: centred in fp64, scaled by 1/(b^2 sigma_L), rounded once
  // (replicate padding comes from the clamped tile rows/cols; halo lanes at
  // the image border see clamped duplicates and are never outputs)
  float Lt[B][B];
  float sumLt;
  {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) s += Ls[wp + r][lane + c];
    const double mu = s / (double)(B * B);
    double ss = 0.0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double dv = Ls[wp + r][lane + c] - mu;
        ss = fma(dv, dv, ss);
      }
    const double sigma = sqrt(ss / (double)(B * B));
    const bool okL = inimg && sigma >= a.sigma_eps;
    const double kL = okL ? 1.0 / ((double)(B * B) * sigma) : 0.0;
    float sl = 0.f;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const float f = (float)((Ls[wp + r][lane + c] - mu) * kL);
        Lt[r][c] = f;
        sl += f;
      }
    sumLt = okL ? sl : qnan;   // NaN: every cost of a flat block is -1
  }

  // ---- prior window (candidates in ascending z, strict '>', init -2)
  bool trusted = false;
  int wlo = 1, whi = 0, zW = 0;
  float bW = -2.f;
  if (a.wc != nullptr && inner) {
    const int c = a.wc[(int64_t)i * a.ldw + j];
    if (c != kWcNone) {
      trusted = true;
      wlo = max(c - a.radius, 0);
      whi = min(c + a.radius, d);
      zW = wlo;
    }
  }

  // all costs beyond zmax are -1 for every pixel of this CTA (exact skip)
  const int zmax = min(d, DIR > 0 ? (x0 + 30) : (W - x0));

  float bF = -2.f, bN = -3.0e38f;
  int zF = 0, zN = 0;

  store(0);
  __syncthreads();
  int cur = 0;
  for (int z0 = 0; z0 <= zmax; z0 += ZC, cur ^= 1) {
    const bool more = z0 + ZC <= zmax;
    if (more) fetch(z0 + ZC);   // in flight during this chunk's math
    const bool wchunk = __any_sync(kFull, trusted && wlo <= z0 + ZC - 1 && whi >= z0);
    int nz;
    if (z0 + ZC - 1 <= zmax) {
      sweep_chunk<B, DIR, ZC, NR, ZC>(Rs[cur], Ms[cur], Hs[cur], Lt, sumLt, z0, 0, zmax,
                                      inimg, lane, wp, bF, zF, wchunk, wlo, whi, bW, zW);
      nz = ZC;
    } else {
      nz = zmax - z0 + 1;
      for (int zo = 0; zo < nz; zo += 4)
        sweep_chunk<B, DIR, ZC, NR, 4>(Rs[cur], Ms[cur], Hs[cur], Lt, sumLt, z0, zo, zmax,
                                       inimg, lane, wp, bF, zF, wchunk, wlo, whi, bW, zW);
    }
    if (more) store(cur ^ 1);
    __syncthreads();
    if (inner) {
      const HsT& hs = Hs[cur];
#pragma unroll
      for (int zz = 0; zz < ZC; ++zz) {
        const float nb = (hs[zz][wp - 1][lane] + hs[zz][wp][lane]) + hs[zz][wp + 1][lane];
        if (zz < nz && nb > bN) { bN = nb; zN = z0 + zz; }
      }
    }
  }

  // ---- epilogue: the reference's gates
  if (trusted && bW == -2.f) { bW = -1.f; zW = wlo; }  // window beyond zmax: all -1
  const int members = ((i > 0) + 1 + (i < H - 1)) * ((j > 0) + 1 + (j < W - 1));
  bool low = false;
  if (a.mode == kSweepPipeline) {
    if (inner) {
      const float cs = trusted ? bW : bF;
      const int zs = trusted ? zW : zF;
      low = (double)cs <= a.alpha;
      const int64_t o = (int64_t)i * a.ldo + j;
      a.dout[o] = (int16_t)(low ? zN : zs);
      a.cout[o] = low ? bN / (float)members : cs;
      a.low[o] = (uint8_t)low;
    }
    const unsigned bal = __ballot_sync(kFull, low && i >= a.rows.cnt_lo && i < a.rows.cnt_hi);
    if (lane == 0 && bal) atomicAdd(&a.counters[kCntRefined], (unsigned long long)__popc(bal));
  } else if (inner) {
    const int64_t o = (int64_t)i * W + j;
    a.fz[o] = (int16_t)zF;
    a.fc[o] = bF;
    if (a.wz) { a.wz[o] = (int16_t)zW; a.wcst[o] = trusted ? bW : -2.f; }
    a.nz[o] = (int16_t)zN;
    a.nc[o] = bN / (float)members;
  }
}

// ---------------------------------------------------------------------------
// Generic fallback for blocks without a register-resident specialisation
// (block > 11): one pixel per thread, window read through L1, fp64 direct
// sums.  Same tile/halo structure and epilogue as the specialised kernel.
template <int DIR, int NR>
__global__ void __launch_bounds__(NR * 32)
sweep_generic(const SweepArgs a) {
  __shared__ float Hs[NR][32];
  const int B = a.block, H2 = B / 2;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 30, y0 = a.rows.lo + blockIdx.y * (NR - 2);
  const int i = y0 - 1 + wp, j = x0 - 1 + lane;
  const int H = a.H, W = a.W, d = a.d;
  const bool inimg = (i >= 0) && (i < H) && (j >= 0) && (j < W);
  const bool inner = inimg && lane >= 1 && lane <= 30 && wp >= 1 && wp <= NR - 2;
  const int ic = clampi(i, 0, H - 1), jc = clampi(j, 0, W - 1);
  double s = 0.0;
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c)
      s += a.Lv(clampi(ic + r - H2, 0, H - 1), clampi(jc + c - H2, 0, W - 1));
  const double mu = s / (double)(B * B);
  double ss = 0.0;
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) {
      const double dv = a.Lv(clampi(ic + r - H2, 0, H - 1), clampi(jc + c - H2, 0, W - 1)) - mu;
      ss += dv * dv;
    }
  const double sigma = sqrt(ss / (double)(B * B));
  int zlim = -1;
  double kL = 0.0;
  if (inimg && sigma >= a.sigma_eps) {
    kL = 1.0 / ((double)(B * B) * sigma);
    zlim = DIR > 0 ? j : (W - 1 - j);
  }
  bool trusted = false;
  int wlo = 1, whi = 0;
  if (a.wc != nullptr && inner) {
    const int c = a.wc[(int64_t)i * a.ldw + j];
    if (c != kWcNone) { trusted = true; wlo = max(c - a.radius, 0); whi = min(c + a.radius, d); }
  }
  float bF = -2.f, bW = -2.f, bN = -3.0e38f;
  int zF = 0, zW = 0, zN = 0;
  for (int z = 0; z <= d; ++z) {
    float rho = -1.f;
    if (z <= zlim) {
      const int q = j - DIR * z;
      const int64_t so = (int64_t)ic * a.lds + q;
      const float is = a.isR[so];
      if (is > 0.f) {
        const double muR = (double)a.muR[so];
        double acc = 0.0;
        for (int r = 0; r < B; ++r) {
          const int yr = clampi(ic + r - H2, 0, H - 1);
          for (int c = 0; c < B; ++c)
            acc += (a.Lv(yr, clampi(jc + c - H2, 0, W - 1)) - mu) *
                   (a.Rv(yr, clampi(q + c - H2, 0, W - 1)) - muR);
        }
        double v = acc * kL * (double)is;
        rho = (float)fmin(fmax(v, -1.0), 1.0);
      }
    }
    if (rho > bF) { bF = rho; zF = z; }
    if (z >= wlo && z <= whi && rho > bW) { bW = rho; zW = z; }
    const float o = inimg ? rho : 0.f;
    const float hl = __shfl_up_sync(kFull, o, 1);
    const float hr = __shfl_down_sync(kFull, o, 1);
    Hs[wp][lane] = (hl + o) + hr;
    __syncthreads();
    if (inner) {
      const float nb = (Hs[wp - 1][lane] + Hs[wp][lane]) + Hs[wp + 1][lane];
      if (nb > bN) { bN = nb; zN = z; }
    }
    __syncthreads();
  }
  const int members = ((i > 0) + 1 + (i < H - 1)) * ((j > 0) + 1 + (j < W - 1));
  bool low = false;
  if (a.mode == kSweepPipeline) {
    if (inner) {
      const float cs = trusted ? bW : bF;
      const int zs = trusted ? zW : zF;
      low = (double)cs <= a.alpha;
      const int64_t o = (int64_t)i * a.ldo + j;
      a.dout[o] = (int16_t)(low ? zN : zs);
      a.cout[o] = low ? bN / (float)members : cs;
      a.low[o] = (uint8_t)low;
    }
    const unsigned bal = __ballot_sync(kFull, low && i >= a.rows.cnt_lo && i < a.rows.cnt_hi);
    if (lane == 0 && bal) atomicAdd(&a.counters[kCntRefined], (unsigned long long)__popc(bal));
  } else if (inner) {
    const int64_t o = (int64_t)i * W + j;
    a.fz[o] = (int16_t)zF;
    a.fc[o] = bF;
    if (a.wz) { a.wz[o] = (int16_t)zW; a.wcst[o] = trusted ? bW : -2.f; }
    a.nz[o] = (int16_t)zN;
    a.nc[o] = bN / (float)members;
  }
}

template <int B, int ZC, int NR>
constexpr size_t sweep_smem() {
  return 2 * sizeof(float[NR + B - 1][30 + B + ZC]) + 2 * sizeof(float2[NR][31 + ZC]) +
         2 * sizeof(float[ZC][NR][32]);
}

template <int B, int DIR, int ZC, int NR, int MINB>
cudaError_t launch_v(const SweepArgs& a, cudaStream_t s) {
  constexpr size_t smem = sweep_smem<B, ZC, NR>();
  static SmemAttr attr;
  if (cudaError_t e = attr.ensure(sweep_kernel<B, DIR, ZC, NR, MINB>, smem); e != cudaSuccess) return e;
  SweepArgs b = a;   // CTA rows on the whole-image grid (see sweep2.cu)
  b.rows.lo = (a.rows.lo / (NR - 2)) * (NR - 2);
  dim3 grid((a.W + 29) / 30, (b.rows.hi - b.rows.lo + NR - 3) / (NR - 2));
  sweep_kernel<B, DIR, ZC, NR, MINB><<<grid, NR * 32, smem, s>>>(b);
  return cudaGetLastError();
}

template <int B, int DIR>
cudaError_t launch_b(const SweepArgs& a, cudaStream_t s) {
  if constexpr (B <= 7) {
    return launch_v<B, DIR, 16, 16, 1>(a, s);
  } else {
    return launch_v<B, DIR, 16, 8, 1>(a, s);
  }
}

template <int DIR>
cudaError_t launch_dir(const SweepArgs& a, cudaStream_t s) {
  switch (a.block) {
    case 3: return launch_b<3, DIR>(a, s);
    case 5: return launch_b<5, DIR>(a, s);
    case 7: return launch_b<7, DIR>(a, s);
    case 9: return launch_b<9, DIR>(a, s);
    case 11: return launch_b<11, DIR>(a, s);
    default: {
      constexpr int NR = 8;
      SweepArgs b = a;
      b.rows.lo = (a.rows.lo / (NR - 2)) * (NR - 2);
      dim3 grid((a.W + 29) / 30, (b.rows.hi - b.rows.lo + NR - 3) / (NR - 2));
      sweep_generic<DIR, NR><<<grid, NR * 32, 0, s>>>(b);
      return cudaGetLastError();
    }
  }
}

}  // namespace

bool sweep_supported_block(int b) { return b >= 3 && (b & 1) && b <= 63; }

namespace {

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
// MSHBM_SWEEP_IMPL: 1 = one pixel per thread (sweep_kernel), 2 = sweep2 (default)
int sweep_impl() {
  static int v = env_int("MSHBM_SWEEP_IMPL", 2);
  return v;
}
// MSHBM_SWEEP4: 0 = sweep2 everywhere, 1 = sweep4 where supported and large
// enough (default), 2 = sweep4 wherever supported (tests)
int sweep4_mode() {
  static int v = env_int("MSHBM_SWEEP4", 1);
  return v;
}
// MSHBM_SWEEP4_GUARD=0 drops the precision guard (measurement only)
bool sweep4_guard() {
  static int v = env_int("MSHBM_SWEEP4_GUARD", 1);
  return v != 0;
}

}  // namespace

bool sweep_uses_sweep4(const SweepArgs& a) {
  return sweep4_mode() != 0 && sweep_impl() >= 2 && sweep4_supported(a, sweep4_mode() == 2);
}

// Tiles the sweep4 precision guard flagged (csrc/stages.cu) are computed by
// sweep2 in fixup mode: it writes and counts only their pixels, and its CTAs
// on unflagged tiles return at once.  It reads what sweep4 reads and writes
// disjoint pixels, so it may run concurrently with sweep4.
cudaError_t launch_sweep4_fixup(const SweepArgs& a, cudaStream_t s) {
  if (!sweep4_guard()) return cudaSuccess;
  SweepArgs b = a;
  b.tile_h = sweep4_th();
  b.fixup = 1;
  return launch_sweep2(b, s);
}

cudaError_t launch_sweep(const SweepArgs& a, cudaStream_t s, int* n_launch) {
  if (n_launch) ++*n_launch;
  const int impl = sweep_impl();
  if (sweep_uses_sweep4(a)) {
    SweepArgs b = a;
    b.tile_h = sweep4_th();
    if (!sweep4_guard()) b.tile_flags = nullptr;
    if (n_launch && a.wc != nullptr) ++*n_launch;   // + prior_select_kernel
    return launch_sweep4(b, s);   // + launch_sweep4_fixup (caller's stream choice)
  }
  if (impl >= 2 && sweep2_supported(a.block)) return launch_sweep2(a, s);
  return a.dir > 0 ? launch_dir<1>(a, s) : launch_dir<-1>(a, s);
}

}  // namespace mshbm
