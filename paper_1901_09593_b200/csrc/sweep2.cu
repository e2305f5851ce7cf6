// Dense fused ZNCC z-sweep, two vertically adjacent pixels per thread.
//
// Same contract as sweep.cu (one launch per level; full-range, prior-window
// and 3x3-summed winner-take-all fused; gates in the epilogue), but each
// thread owns pixels A = (i, j) and B = (i+1, j).  Their windows share b-1
// rows, so with P(z) = sum over the shared rows of (L - muA)(R - c):
//   S_A(z) = P(z) + row_top(z)
//   S_B(z) = P(z) + row_bottom(z) + b^2 (muA - muB) * (muR_B(q) - c)
// where both extra rows are centred by muA; the last term re-centres B's
// whole window from muA to muB exactly (sum over a window of (R - c) is
// b^2 (muR - c)).  That is b^2 + b + 1 FMAs per two pixels instead of 2 b^2,
// and every staged right-image row feeds both pixels.
//
// Reference semantics: matcher.py:184-193 (full search), 263-320 (prior
// window), 196-233 (3x3-summed refinement); zncc.py:271-287 (cost).
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mshbm {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ float fma_sat(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
template <int B, int ZC, int NR>
struct Sweep2Smem {
  static constexpr int NROW = 2 * NR;
  static constexpr int RW = (30 + B + ZC + 1) & ~1;   // staged strip row length
  static constexpr int RR = NROW + B - 1;
  static constexpr int SW = 31 + ZC;
  static constexpr int LC = 31 + B;
  using RsT = float[RR][RW];
  using MsT = float2[NROW][SW];
  using HxT = float[ZC][2][NR][32];   // [0] hsA, [1] hsB (horizontal 3-sums)
  using LsT = double[RR][LC];
  static constexpr int NRS = 2;   // strip buffers (double-buffered)
  static constexpr size_t bytes() {
    return NRS * sizeof(RsT) + 2 * sizeof(MsT) + 2 * sizeof(HxT);
  }
};

// One chunk of NZ disparities (NZ == ZC, or 4 for the tail) for pixels A, B.
template <int B, int DIR, int ZC, int NR, int NZ>
__device__ __forceinline__ void chunk2(
    const typename Sweep2Smem<B, ZC, NR>::RsT& Rs,
    const typename Sweep2Smem<B, ZC, NR>::MsT& Ms,
    typename Sweep2Smem<B, ZC, NR>::HxT& Hx, const float (&Lt)[B][B], const float (&Lb)[B],
    float kLA, float kLB, float dW, int z0, int zoff, int zend, bool inA, bool inB, int lane,
    int wp, float (&best)[4], int (&bestz)[4], bool wchunk, const int (&wlo)[2],
    const int (&whi)[2]) {
  float SA[NZ], P[NZ];
  {
#pragma unroll
    for (int zz = 0; zz < NZ; ++zz) SA[zz] = 0.f, P[zz] = 0.f;
    // window rows r = 0 (A only), 1..B-1 (shared), B (B's bottom)
#pragma unroll
    for (int r = 0; r <= B; ++r) {
      const float* rp = &Rs[2 * wp + r][lane];
#pragma unroll
      for (int e = 0; e < NZ + B - 1; ++e) {
        const int eo = DIR > 0 ? (ZC - NZ - zoff) + e : zoff + e;
        const float v = rp[eo];
#pragma unroll
        for (int c = 0; c < B; ++c) {
          const int g = e - c;
          if (g >= 0 && g < NZ) {
            const int zz = DIR > 0 ? (NZ - 1 - g) : g;
            if (r == 0) SA[zz] = fmaf(Lt[0][c], v, SA[zz]);
            else if (r < B) P[zz] = fmaf(Lt[r][c], v, P[zz]);
            else P[zz] = fmaf(Lb[c], v, P[zz]);
          }
        }
      }
      if (r == B - 1) {
#pragma unroll
        for (int zz = 0; zz < NZ; ++zz) SA[zz] += P[zz];   // S_A complete
      }
    }
  }
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) {
    const int z = z0 + zoff + zz;
    const int g = DIR > 0 ? (ZC - 1 - (zoff + zz)) : (zoff + zz);
    const float2 ma = Ms[2 * wp][lane + g];       // (muR - c, 0.5/sigma_R or NaN)
    const float2 mb = Ms[2 * wp + 1][lane + g];
    // half-range cost c' = sat(c/2 + 1/2) in [0, 1]: the clamp of c to
    // [-1, 1] is the .sat modifier, and NaN (degenerate or out-of-image
    // blocks, right centre outside the image) saturates to 0, i.e. c = -1.
    // Pixels outside the image also come out as 0, the neutral element of
    // the 3x3 sums.
    float ra = fma_sat(SA[zz] * kLA, ma.y, 0.5f);
    float rb = fma_sat(fmaf(dW, mb.x, P[zz]) * kLB, mb.y, 0.5f);
    if (NZ < ZC && z > zend) ra = -3.f, rb = -3.f;  // masked tail slot
    if (ra > best[0]) { best[0] = ra; bestz[0] = z; }
    if (rb > best[1]) { best[1] = rb; bestz[1] = z; }
    if (wchunk) {
      if (z >= wlo[0] && z <= whi[0] && ra > best[2]) { best[2] = ra; bestz[2] = z; }
      if (z >= wlo[1] && z <= whi[1] && rb > best[3]) { best[3] = rb; bestz[3] = z; }
    }
    // (masked tail slots carry -3 into sums the nb pass never reads)
    const float ha = (__shfl_up_sync(kFull, ra, 1) + ra) + __shfl_down_sync(kFull, ra, 1);
    const float hb = (__shfl_up_sync(kFull, rb, 1) + rb) + __shfl_down_sync(kFull, rb, 1);
    Hx[zoff + zz][0][wp][lane] = ha;
    Hx[zoff + zz][1][wp][lane] = hb;
  }
}

template <int B, int DIR, int ZC, int NR, int MINB>
__device__ __forceinline__ void sweep2_body(const SweepArgs& a, const int bx, const int by) {
  using SM = Sweep2Smem<B, ZC, NR>;
  constexpr int H2 = B / 2;
  constexpr int NT = NR * 32;
  constexpr int NROW = SM::NROW, RW = SM::RW, RR = SM::RR, SW = SM::SW, LC = SM::LC;
  extern __shared__ float4 smem4[];
  typename SM::RsT* Rs = reinterpret_cast<typename SM::RsT*>(smem4);
  typename SM::MsT* Ms = reinterpret_cast<typename SM::MsT*>(Rs + SM::NRS);
  typename SM::HxT* Hx = reinterpret_cast<typename SM::HxT*>(Ms + 2);

  const int lane = threadIdx.x & 31;
  const int wp = threadIdx.x >> 5;
  const int x0 = bx * 30;
  const int y0 = a.rows.lo + by * (NROW - 2);
  const int iA = y0 - 1 + 2 * wp, iB = iA + 1;
  const int j = x0 - 1 + lane;
  const int H = a.H, W = a.W, d = a.d;
  const bool colin = j >= 0 && j < W;
  const bool inA = colin && iA >= 0 && iA < H;
  const bool inB = colin && iB >= 0 && iB < H;
  const bool lanein = lane >= 1 && lane <= 30;
  const bool innerA = inA && lanein && wp >= 1;
  const bool innerB = inB && lanein && wp <= NR - 2;
  const float qnan = __int_as_float(0x7fc00000);
  // sweep4 fixup: only pixels of the tiles sweep4's precision guard flagged
  auto flagged = [&](int i, int jj) {
    return a.tile_flags[(int64_t)tile_row(i, a.tile_h) * a.flags_ld + jj / 16] != 0;
  };
  if (a.fixup) {
    const int ilo = max(y0, 0), ihi = min(y0 + NROW - 3, H - 1);
    const int jlo = max(x0, 0), jhi = min(x0 + 29, W - 1);
    bool any = false;
    for (int ti = tile_row(ilo, a.tile_h); ti <= tile_row(ihi, a.tile_h) && !any; ++ti)
      for (int tj = jlo / 16; tj <= jhi / 16; ++tj)
        any |= a.tile_flags[(int64_t)ti * a.flags_ld + tj] != 0;
    if (!any || ilo > ihi || jlo > jhi) return;   // uniform over the CTA
  }

  // ---- staging: cp.async from the padded fp32 arrays (prep_staging) straight
  // into the double-buffered strip; no clamps on columns, no conversion, no
  // prefetch registers.  Warp w copies rows w, w+NR, ...
  const float* __restrict__ Rp = a.Rp + a.pc;
  const float2* __restrict__ Mp = a.Mp + a.pc;
  // per-thread source offsets of the rows this warp copies, computed once
  // (row clamp, pitch multiply, lane); each chunk only adds its z shift
  constexpr int KR = (RR + NR - 1) / NR, KM = (NROW + NR - 1) / NR;
  constexpr int UR = (RW + 31) / 32, UM = (SW + 31) / 32;
  // Kept in registers, except at b = 7 (2 CTAs at the 128-register cap,
  // where they would spill): there in shared memory, warp-uniform broadcast
  // loads, no registers held across the sweep (measured best per b).
  constexpr bool kOffReg = (B != 7);
  constexpr int KO = KR + KM;
  __shared__ int s_off[kOffReg ? 1 : NR][KO];
  int r_off[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k)
    r_off[k] = k < KR
        ? clampi(y0 - 1 - H2 + wp + NR * k, 0, H - 1) * (int)a.ldp + (x0 - 1 - H2)
        : clampi(y0 - 1 + wp + NR * (k - KR), 0, H - 1) * (int)a.ldp + (x0 - 1);
  if constexpr (!kOffReg) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < KO; ++k) s_off[wp][k] = r_off[k];
    }
    __syncwarp();
  }
  auto off = [&](int k) { return kOffReg ? r_off[k] : s_off[wp][k]; };
  auto issue = [&](int buf, int z0) {
    const int zs = (DIR > 0 ? (-z0 - (ZC - 1)) : z0) + lane;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int rr = wp + NR * k;
      if (rr < RR) {
        const float* src = Rp + (off(k) + zs);
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int e = lane + 32 * u;
          if (e < RW) {
            cp_async4(&Rs[buf][rr][e], src + 32 * u);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      const int rr = wp + NR * k;
      if (rr < NROW) {
        const float2* src = Mp + (off(KR + k) + zs);
#pragma unroll
        for (int u = 0; u < UM; ++u) {
          const int e = lane + 32 * u;
          if (e < SW) cp_async8(&Ms[buf][rr][e], src + 32 * u);
        }
      }
    }
    cp_async_commit();
  };
  issue(0, 0);

  // ---- left tile (fp64) through shared memory (aliases Hx, written later)
  using LsT = typename SM::LsT;
  static_assert(sizeof(LsT) <= 2 * sizeof(typename SM::HxT), "left tile must fit");
  LsT& Ls = *reinterpret_cast<LsT*>(Hx);
  {
    // all loads in flight before the stores (one memory latency, not NL)
    constexpr int NL = (RR * LC + NT - 1) / NT;
    double v[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int t = threadIdx.x + NT * k;
      const int rr = t / LC, e = t - rr * LC;
      v[k] = t < RR * LC ? a.Lv(clampi(y0 - 1 - H2 + rr, 0, H - 1), clampi(x0 - 1 - H2 + e, 0, W - 1))
                         : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int t = threadIdx.x + NT * k;
      const int rr = t / LC, e = t - rr * LC;
      if (t < RR * LC) Ls[rr][e] = v[k];
    }
  }
  __syncthreads();

  // ---- left windows: A centred by muA (rows 0..B-1), B's bottom row by muA
  float Lt[B][B], Lb[B];
  float kLA, kLB, dW;
  {
    const int r0 = 2 * wp;
    double sA = 0.0, top = 0.0, bot = 0.0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) sA += Ls[r0 + r][lane + c];
#pragma unroll
    for (int c = 0; c < B; ++c) top += Ls[r0][lane + c], bot += Ls[r0 + B][lane + c];
    const double muA = sA / (double)(B * B);
    const double muB = (sA - top + bot) / (double)(B * B);
    double ssA = 0.0, ssB = 0.0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double v = Ls[r0 + r][lane + c];
        const double da = v - muA;
        ssA = fma(da, da, ssA);
        Lt[r][c] = (float)da;
      }
#pragma unroll
    for (int r = 1; r <= B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double db = Ls[r0 + r][lane + c] - muB;
        ssB = fma(db, db, ssB);
      }
#pragma unroll
    for (int c = 0; c < B; ++c) Lb[c] = (float)(Ls[r0 + B][lane + c] - muA);
    const double sgA = sqrt(ssA / (double)(B * B)), sgB = sqrt(ssB / (double)(B * B));
    kLA = (inA && sgA >= a.sigma_eps) ? (float)(1.0 / ((double)(B * B) * sgA)) : qnan;
    kLB = (inB && sgB >= a.sigma_eps) ? (float)(1.0 / ((double)(B * B) * sgB)) : qnan;
    dW = (float)((double)(B * B) * (muA - muB));
  }

  // ---- prior windows of A and B
  bool trusted[2] = {false, false};
  int wlo[2] = {1, 1}, whi[2] = {0, 0};
  if (a.wc != nullptr) {
    const bool inn[2] = {innerA, innerB};
    const int ii[2] = {iA, iB};
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      if (inn[p]) {
        const int c = a.wc[(int64_t)ii[p] * a.ldw + j];
        if (c != kWcNone) {
          trusted[p] = true;
          wlo[p] = max(c - a.radius, 0);
          whi[p] = min(c + a.radius, d);
        }
      }
    }
  }

  const int zmax = min(d, DIR > 0 ? (x0 + 30) : (W - x0));
  // best[0..1]: full range A/B, best[2..3]: window A/B; nbv/nbz: 3x3 sums
  float best[4] = {-2.f, -2.f, -2.f, -2.f};
  int bestz[4] = {0, 0, wlo[0], wlo[1]};
  float nbv[2] = {-3.0e38f, -3.0e38f};
  int nbz[2] = {0, 0};

  cp_async_wait_all();
  __syncthreads();
  int cur = 0;
  for (int z0 = 0; z0 <= zmax; z0 += ZC, cur ^= 1) {
    const bool more = z0 + ZC <= zmax;
    if (more) issue(cur ^ 1, z0 + ZC);   // lands during this chunk's math
    const bool wchunk = __any_sync(kFull, (trusted[0] && wlo[0] <= z0 + ZC - 1 && whi[0] >= z0) ||
                                             (trusted[1] && wlo[1] <= z0 + ZC - 1 && whi[1] >= z0));
    int nz;
    if (z0 + ZC - 1 <= zmax) {
      chunk2<B, DIR, ZC, NR, ZC>(Rs[cur], Ms[cur], Hx[cur], Lt, Lb, kLA, kLB, dW, z0, 0, zmax,
                                 inA, inB, lane, wp, best, bestz, wchunk, wlo, whi);
      nz = ZC;
    } else {
      nz = zmax - z0 + 1;
      for (int zo = 0; zo < nz; zo += 4)
        chunk2<B, DIR, ZC, NR, 4>(Rs[cur], Ms[cur], Hx[cur], Lt, Lb, kLA, kLB, dW, z0, zo, zmax,
                                  inA, inB, lane, wp, best, bestz, wchunk, wlo, whi);
    }
    cp_async_wait_all();
    __syncthreads();
    // vertical 3-sums: A = B(above) + (A + B), B = (A + B) + A(below); the
    // edge warps' out-of-tile reads are clamped and never used (innerA/B)
    const typename SM::HxT& hx = Hx[cur];
    const int wu = wp > 0 ? wp - 1 : 0, wd = wp < NR - 1 ? wp + 1 : NR - 1;
#pragma unroll
    for (int zz = 0; zz < ZC; ++zz) {
      const float t = hx[zz][0][wp][lane] + hx[zz][1][wp][lane];
      const float nba = hx[zz][1][wu][lane] + t;
      const float nbb = t + hx[zz][0][wd][lane];
      if (innerA && zz < nz && nba > nbv[0]) { nbv[0] = nba; nbz[0] = z0 + zz; }
      if (innerB && zz < nz && nbb > nbv[1]) { nbv[1] = nbb; nbz[1] = z0 + zz; }
    }
  }

  // ---- epilogue: the reference's gates, per pixel
  const bool inner[2] = {innerA, innerB};
  const int ii[2] = {iA, iB};
  unsigned nlow = 0;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int i = ii[p];
    const int members = ((i > 0) + 1 + (i < H - 1)) * ((j > 0) + 1 + (j < W - 1));
    // back from half-range c' to c = 2c' - 1 (exact for c' >= 1/4)
    float bw = best[2 + p];
    bw = (trusted[p] && bw == -2.f) ? -1.f : 2.f * bw - 1.f;   // window beyond zmax: all -1
    const float bf = 2.f * best[p] - 1.f;
    const float nbc = 2.f * nbv[p] / (float)members - 1.f;
    bool low = false;
    if (a.mode == kSweepPipeline) {
      if (inner[p] && (!a.fixup || flagged(i, j))) {
        const float cs = trusted[p] ? bw : bf;
        const int zs = trusted[p] ? bestz[2 + p] : bestz[p];
        low = (double)cs <= a.alpha;
        const int64_t o = (int64_t)i * a.ldo + j;
        a.dout[o] = (int16_t)(low ? nbz[p] : zs);
        a.cout[o] = low ? nbc : cs;
        a.low[o] = (uint8_t)low;
      }
      nlow += (low && i >= a.rows.cnt_lo && i < a.rows.cnt_hi) ? 1u : 0u;
    } else if (inner[p]) {
      const int64_t o = (int64_t)i * W + j;
      a.fz[o] = (int16_t)bestz[p];
      a.fc[o] = bf;
      if (a.wz) { a.wz[o] = (int16_t)bestz[2 + p]; a.wcst[o] = trusted[p] ? bw : -2.f; }
      a.nz[o] = (int16_t)nbz[p];
      a.nc[o] = nbc;
    }
  }
  if (a.mode == kSweepPipeline) {
    const int slot[1] = {kCntRefined};
    const unsigned long long val[1] = {nlow};
    const bool mx[1] = {false};
    block_accumulate<1>(a.counters, slot, val, mx);
  }
}

// One CTA per 30 x (2 NR - 2) job; in sweep4-fixup list mode a persistent
// grid walks the job list the list kernel built (only jobs that touch
// guard-flagged tiles), so an empty list costs one short wave.
template <int B, int DIR, int ZC, int NR, int MINB>
__global__ void __launch_bounds__(NR * 32, MINB) sweep2_kernel(const SweepArgs a) {
  pdl_wait();
  // one inlined copy of the body (instruction cache): the plain launch is a
  // one-iteration loop over its own block
  const bool lm = a.fixup && a.fix_list != nullptr;
  const int n = lm ? *a.fix_count : 1;
  for (int i = lm ? (int)blockIdx.x : 0; i < n; i += lm ? (int)gridDim.x : 1) {
    int bx = blockIdx.x, by = blockIdx.y;
    if (lm) {
      const int job = a.fix_list[i];
      bx = job % a.fix_nbx;
      by = job / a.fix_nbx;
    }
    sweep2_body<B, DIR, ZC, NR, MINB>(a, bx, by);
    if (lm) __syncthreads();   // shared memory is reused by the next job
  }
}

// sweep2 job geometry: NR warps x 2 pixel rows (NROW - 2 output rows per
// job), NR = 16 at b = 5 and 8 otherwise (launch_fixup_list reads this too).
constexpr int sweep2_nr(int b) { return b == 5 ? 16 : 8; }

template <int B, int DIR, int ZC, int NR, int MINB>
cudaError_t launch2(const SweepArgs& a, cudaStream_t s) {
  static_assert(NR == sweep2_nr(B), "job geometry shared with launch_fixup_list");
  constexpr size_t smem = Sweep2Smem<B, ZC, NR>::bytes();
  static SmemAttr attr;
  cudaError_t e = attr.ensure(sweep2_kernel<B, DIR, ZC, NR, MINB>, smem);
  if (e != cudaSuccess) return e;
  constexpr int NROW = 2 * NR;
  // CTA rows stay on the whole-image grid (row bands are then bit-identical:
  // the per-CTA offset c of the right strip depends on the CTA)
  SweepArgs b = a;
  b.rows.lo = (a.rows.lo / (NROW - 2)) * (NROW - 2);
  dim3 grid((a.W + 29) / 30, (b.rows.hi - b.rows.lo + NROW - 3) / (NROW - 2));
  if (b.fixup && b.fix_list != nullptr) {   // persistent grid over the fixup job list
    b.fix_nbx = grid.x;
    grid = dim3(std::min<unsigned>(grid.x * grid.y, 2 * 148), 1);
  }
  return launch_pdl(sweep2_kernel<B, DIR, ZC, NR, MINB>, grid, dim3(NR * 32), smem, s, b);
}

template <int DIR>
cudaError_t launch2_dir(const SweepArgs& a, cudaStream_t s) {
  switch (a.block) {
    case 3: return launch2<3, DIR, 16, 8, 2>(a, s);
    case 5: return launch2<5, DIR, 16, 16, 1>(a, s);
    case 7: return launch2<7, DIR, 16, 8, 2>(a, s);
    case 9: return launch2<9, DIR, 16, 8, 1>(a, s);
    case 11: return launch2<11, DIR, 16, 8, 1>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// sweep4 fixup job list: the sweep2 jobs (30 columns x 2 NR - 2 rows,
// NR = sweep2_nr(b), the geometry launch2 uses) whose output
// pixels touch a tile the sweep4 guard flagged.  One thread per job; *count
// is zeroed with the flags before every run.
__global__ void __launch_bounds__(256) fixup_list_kernel(const unsigned* flags, int64_t flags_ld,
                                                         int tile_h, int h, int w, int lo,
                                                         int job_rows, int nbx, int nby,
                                                         int* list, int* count) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nbx * nby) return;
  const int bx = j % nbx, by = j / nbx;
  const int y0 = lo + by * job_rows, x0 = bx * 30;
  const int ilo = max(y0, 0), ihi = min(y0 + job_rows - 1, h - 1);
  const int jlo = x0, jhi = min(x0 + 29, w - 1);
  bool any = false;
  for (int ti = tile_row(ilo, tile_h); ti <= tile_row(ihi, tile_h) && !any; ++ti)
    for (int tj = jlo / 16; tj <= jhi / 16; ++tj) any |= flags[(int64_t)ti * flags_ld + tj] != 0;
  if (any && ilo <= ihi && jlo <= jhi) list[atomicAdd(count, 1)] = j;
}

cudaError_t launch_fixup_list(const unsigned* flags, int64_t flags_ld, int tile_h, int h, int w,
                              RowBand rows, int block, int* list, int* count, cudaStream_t s) {
  const int nr = sweep2_nr(block);
  const int job_rows = 2 * nr - 2;
  const int lo = (rows.lo / job_rows) * job_rows;
  const int nbx = (w + 29) / 30, nby = std::max((rows.hi - lo + job_rows - 1) / job_rows, 0);
  if (nbx * nby == 0) return cudaSuccess;
  fixup_list_kernel<<<(nbx * nby + 255) / 256, 256, 0, s>>>(flags, flags_ld, tile_h, h, w, lo,
                                                           job_rows, nbx, nby, list, count);
  return cudaGetLastError();
}

bool sweep2_supported(int b) { return b == 3 || b == 5 || b == 7 || b == 9 || b == 11; }

cudaError_t launch_sweep2(const SweepArgs& a, cudaStream_t s) {
  return a.dir > 0 ? launch2_dir<1>(a, s) : launch2_dir<-1>(a, s);
}

}  // namespace mshbm
