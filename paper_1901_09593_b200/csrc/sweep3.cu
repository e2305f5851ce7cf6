// Dense fused ZNCC z-sweep, three vertically adjacent pixels per thread.
//
// Same contract as sweep2.cu (one launch per level; full-range, prior-window
// and 3x3-summed winner-take-all fused; gates in the epilogue).  Thread
// (lane, warp) owns pixels P0, P1, P2 = rows i, i+1, i+2 of column j.  Their
// windows cover B+2 image rows; with every row centred by mu0 and
// D_r(z) = sum_c (L[r][c] - mu0) (R[r][q+c] - c) the row dot products,
//   S0 = C + D_0 + D_1
//   S1 = C + D_1 + D_B     + b^2 (mu0 - mu1) (muR(q1) - c)
//   S2 = C + D_B + D_{B+1} + b^2 (mu0 - mu2) (muR(q2) - c)
// with C = D_2 + ... + D_{B-1} shared by all three.  That is (B+2) B FMAs
// plus 8 adds per three pixels (23.7 per pixel at b = 7, against 28.5 for
// two pixels per thread), and P1's 3x3 sum needs no exchange: its upper and
// lower neighbours are P0 and P2 of the same thread.
//
// Measured (C2 level 0, b = 7): 5% fewer instructions than sweep2 but the
// same time (0.73 ms): 12 resident warps per SM instead of 16 and twice the
// chunk overhead at ZC = 8 (ZC = 16 spills at the 168-register cap).  Kept
// as an opt-in (MSHBM_SWEEP_IMPL=3); sweep2 is the default.
//
// Reference semantics: matcher.py:184-193 (full search), 263-320 (prior
// window), 196-233 (3x3-summed refinement); zncc.py:271-287 (cost).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace mshbm {

namespace {

constexpr unsigned kFull3 = 0xffffffffu;

__device__ __forceinline__ void cp_async4_3(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async8_3(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ float fma_sat3(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int B, int ZC, int NR>
struct Sweep3Smem {
  static constexpr int NROW = 3 * NR;
  static constexpr int RW = (30 + B + ZC + 1) & ~1;
  static constexpr int RR = NROW + B - 1;
  static constexpr int SW = 31 + ZC;
  static constexpr int LC = 31 + B;
  using RsT = float[RR][RW];
  using MsT = float2[NROW][SW];
  using HxT = float[ZC][3][NR][32];   // horizontal 3-sums of P0, P1, P2
  using LsT = double[RR][LC];
  static constexpr size_t bytes() {
    return 2 * sizeof(RsT) + 2 * sizeof(MsT) + 2 * sizeof(HxT);
  }
};

// Per-thread state of the three pixels.
struct Px3 {
  float best[3], bw[3], nbv[3];
  int bestz[3], bwz[3], nbz[3], wlo[3], whi[3];
};

// One sub-chunk of NZ disparities (NZ divides ZC; 4 for the tail).
template <int B, int DIR, int ZC, int NR, int NZ>
__device__ __forceinline__ void chunk3(
    const typename Sweep3Smem<B, ZC, NR>::RsT& Rs, const typename Sweep3Smem<B, ZC, NR>::MsT& Ms,
    typename Sweep3Smem<B, ZC, NR>::HxT& Hx, const float (&Lw)[B + 2][B], const float (&kL)[3],
    const float (&dW)[3], int z0, int zoff, int zend, int lane, int wp, bool inner1,
    Px3& st, bool wchunk) {
  float C[NZ], T0[NZ], T1[NZ], TB[NZ], TB1[NZ];
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) C[zz] = T0[zz] = T1[zz] = TB[zz] = TB1[zz] = 0.f;
#pragma unroll
  for (int r = 0; r < B + 2; ++r) {
    const float* rp = &Rs[3 * wp + r][lane];
#pragma unroll
    for (int e = 0; e < NZ + B - 1; ++e) {
      const int eo = DIR > 0 ? (ZC - NZ - zoff) + e : zoff + e;
      const float v = rp[eo];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const int g = e - c;
        if (g >= 0 && g < NZ) {
          const int zz = DIR > 0 ? (NZ - 1 - g) : g;
          const float w = Lw[r][c];
          if (r == 0) T0[zz] = fmaf(w, v, T0[zz]);
          else if (r == 1) T1[zz] = fmaf(w, v, T1[zz]);
          else if (r == B) TB[zz] = fmaf(w, v, TB[zz]);
          else if (r == B + 1) TB1[zz] = fmaf(w, v, TB1[zz]);
          else C[zz] = fmaf(w, v, C[zz]);
        }
      }
    }
  }
#pragma unroll
  for (int zz = 0; zz < NZ; ++zz) {
    const int z = z0 + zoff + zz;
    const int g = DIR > 0 ? (ZC - 1 - (zoff + zz)) : (zoff + zz);
    const float2 m0 = Ms[3 * wp][lane + g];       // (muR - c, 0.5/sigma_R or NaN)
    const float2 m1 = Ms[3 * wp + 1][lane + g];
    const float2 m2 = Ms[3 * wp + 2][lane + g];
    const float s0 = (C[zz] + T1[zz]) + T0[zz];
    const float s1 = (C[zz] + T1[zz]) + TB[zz];
    const float s2 = (C[zz] + TB[zz]) + TB1[zz];
    // half-range cost c' = sat(c/2 + 1/2): clamp, NaN validity and
    // out-of-image masking in one instruction (see sweep2.cu)
    float r[3];
    r[0] = fma_sat3(s0 * kL[0], m0.y, 0.5f);
    r[1] = fma_sat3(fmaf(dW[1], m1.x, s1) * kL[1], m1.y, 0.5f);
    r[2] = fma_sat3(fmaf(dW[2], m2.x, s2) * kL[2], m2.y, 0.5f);
    const bool live = NZ == ZC || z <= zend;
    if (!live) r[0] = r[1] = r[2] = -3.f;   // masked tail slot
#pragma unroll
    for (int p = 0; p < 3; ++p)
      if (r[p] > st.best[p]) { st.best[p] = r[p]; st.bestz[p] = z; }
    if (wchunk) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
        if (z >= st.wlo[p] && z <= st.whi[p] && r[p] > st.bw[p]) { st.bw[p] = r[p]; st.bwz[p] = z; }
    }
    float hs[3];
#pragma unroll
    for (int p = 0; p < 3; ++p)
      hs[p] = (__shfl_up_sync(kFull3, r[p], 1) + r[p]) + __shfl_down_sync(kFull3, r[p], 1);
    // P1's vertical neighbours are P0 and P2 of this thread
    const float nb1 = (hs[0] + hs[1]) + hs[2];
    if (inner1 && live && nb1 > st.nbv[1]) { st.nbv[1] = nb1; st.nbz[1] = z; }
#pragma unroll
    for (int p = 0; p < 3; ++p) Hx[zoff + zz][p][wp][lane] = hs[p];
  }
}

template <int B, int DIR, int ZC, int NR, int NZ, int MINB>
__global__ void __launch_bounds__(NR * 32, MINB)
sweep3_kernel(const SweepArgs a) {
  using SM = Sweep3Smem<B, ZC, NR>;
  constexpr int H2 = B / 2;
  constexpr int NT = NR * 32;
  constexpr int NROW = SM::NROW, RW = SM::RW, RR = SM::RR, SW = SM::SW, LC = SM::LC;
  static_assert(ZC % NZ == 0 && ZC % 4 == 0, "sub-chunking");
  extern __shared__ float4 smem4[];
  typename SM::RsT* Rs = reinterpret_cast<typename SM::RsT*>(smem4);
  typename SM::MsT* Ms = reinterpret_cast<typename SM::MsT*>(Rs + 2);
  typename SM::HxT* Hx = reinterpret_cast<typename SM::HxT*>(Ms + 2);

  const int lane = threadIdx.x & 31;
  const int wp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 30;
  const int y0 = a.rows.lo + blockIdx.y * (NROW - 2);
  const int i0 = y0 - 1 + 3 * wp;     // rows of P0, P1, P2: i0, i0+1, i0+2
  const int j = x0 - 1 + lane;
  const int H = a.H, W = a.W, d = a.d;
  const bool colin = j >= 0 && j < W;
  const bool lanein = lane >= 1 && lane <= 30;
  bool in[3], inner[3];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    in[p] = colin && i0 + p >= 0 && i0 + p < H;
    inner[p] = in[p] && lanein;
  }
  inner[0] = inner[0] && wp >= 1;        // CTA top halo row
  inner[2] = inner[2] && wp <= NR - 2;   // CTA bottom halo row
  const float qnan = __int_as_float(0x7fc00000);

  // ---- staging (as sweep2): cp.async from the padded fp32 arrays
  const float* __restrict__ Rp = a.Rp + a.pc;
  const float2* __restrict__ Mp = a.Mp + a.pc;
  auto issue = [&](int buf, int z0) {
    const int s0 = DIR > 0 ? (x0 - 1 - H2 - z0 - (ZC - 1)) : (x0 - 1 - H2 + z0);
    for (int rr = wp; rr < RR; rr += NR) {
      const float* src = Rp + (int64_t)clampi(y0 - 1 - H2 + rr, 0, H - 1) * a.ldp + s0;
      for (int e = lane; e < RW; e += 32) cp_async4_3(&Rs[buf][rr][e], src + e);
    }
    const int q0 = DIR > 0 ? (x0 - 1 - z0 - (ZC - 1)) : (x0 - 1 + z0);
    for (int rr = wp; rr < NROW; rr += NR) {
      const float2* src = Mp + (int64_t)clampi(y0 - 1 + rr, 0, H - 1) * a.ldp + q0;
      for (int e = lane; e < SW; e += 32) cp_async8_3(&Ms[buf][rr][e], src + e);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  issue(0, 0);

  // ---- left tile (fp64) through shared memory (aliases Hx, written later)
  using LsT = typename SM::LsT;
  static_assert(sizeof(LsT) <= 2 * sizeof(typename SM::HxT), "left tile must fit");
  LsT& Ls = *reinterpret_cast<LsT*>(Hx);
  {
    constexpr int NL = (RR * LC + NT - 1) / NT;
    double v[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int t = threadIdx.x + NT * k;
      const int rr = t / LC, e = t - rr * LC;
      v[k] = t < RR * LC ? a.L[(int64_t)clampi(y0 - 1 - H2 + rr, 0, H - 1) * a.ld +
                              clampi(x0 - 1 - H2 + e, 0, W - 1)]
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

  // ---- left windows: rows 0..B+1 centred by mu0; per-pixel scale and shift
  float Lw[B + 2][B];
  float kL[3], dW[3];
  {
    const int r0 = 3 * wp;
    double rs[B + 2];
#pragma unroll
    for (int r = 0; r < B + 2; ++r) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < B; ++c) t += Ls[r0 + r][lane + c];
      rs[r] = t;
    }
    constexpr double inv = 1.0 / (double)(B * B);
    double mu[3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < B; ++r) t += rs[p + r];
      mu[p] = t * inv;
    }
    double ss[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < B + 2; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double v = Ls[r0 + r][lane + c];
        Lw[r][c] = (float)(v - mu[0]);
#pragma unroll
        for (int p = 0; p < 3; ++p)
          if (r >= p && r < p + B) {
            const double dv = v - mu[p];
            ss[p] = fma(dv, dv, ss[p]);
          }
      }
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double sg = sqrt(ss[p] * inv);
      kL[p] = (in[p] && sg >= a.sigma_eps) ? (float)(1.0 / ((double)(B * B) * sg)) : qnan;
      dW[p] = (float)((double)(B * B) * (mu[0] - mu[p]));
    }
  }

  // ---- prior windows
  Px3 st;
  bool trusted[3] = {false, false, false};
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    st.best[p] = -2.f; st.bw[p] = -2.f; st.nbv[p] = -3.0e38f;
    st.bestz[p] = 0; st.nbz[p] = 0;
    st.wlo[p] = 1; st.whi[p] = 0;
    if (a.wc != nullptr && inner[p]) {
      const int c = a.wc[(int64_t)(i0 + p) * a.ldw + j];
      if (c != kWcNone) {
        trusted[p] = true;
        st.wlo[p] = max(c - a.radius, 0);
        st.whi[p] = min(c + a.radius, d);
      }
    }
    st.bwz[p] = st.wlo[p];
  }

  const int zmax = min(d, DIR > 0 ? (x0 + 30) : (W - x0));
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  int cur = 0;
  for (int z0 = 0; z0 <= zmax; z0 += ZC, cur ^= 1) {
    const bool more = z0 + ZC <= zmax;
    if (more) issue(cur ^ 1, z0 + ZC);   // lands during this chunk's math
    bool wv = false;
#pragma unroll
    for (int p = 0; p < 3; ++p) wv |= trusted[p] && st.wlo[p] <= z0 + ZC - 1 && st.whi[p] >= z0;
    const bool wchunk = __any_sync(kFull3, wv);
    int nz;
    if (z0 + ZC - 1 <= zmax) {
#pragma unroll
      for (int zo = 0; zo < ZC; zo += NZ)
        chunk3<B, DIR, ZC, NR, NZ>(Rs[cur], Ms[cur], Hx[cur], Lw, kL, dW, z0, zo, zmax, lane, wp,
                                   inner[1], st, wchunk);
      nz = ZC;
    } else {
      nz = zmax - z0 + 1;
      for (int zo = 0; zo < nz; zo += 4)
        chunk3<B, DIR, ZC, NR, 4>(Rs[cur], Ms[cur], Hx[cur], Lw, kL, dW, z0, zo, zmax, lane, wp,
                                  inner[1], st, wchunk);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // P0 and P2: vertical neighbours from the warps above / below (clamped
    // indices at the CTA edges are never used: inner[0] / inner[2])
    const typename SM::HxT& hx = Hx[cur];
    const int wu = wp > 0 ? wp - 1 : 0, wd = wp < NR - 1 ? wp + 1 : NR - 1;
#pragma unroll
    for (int zz = 0; zz < ZC; ++zz) {
      const float h1 = hx[zz][1][wp][lane];
      const float nb0 = (hx[zz][2][wu][lane] + hx[zz][0][wp][lane]) + h1;
      const float nb2 = (h1 + hx[zz][2][wp][lane]) + hx[zz][0][wd][lane];
      if (inner[0] && zz < nz && nb0 > st.nbv[0]) { st.nbv[0] = nb0; st.nbz[0] = z0 + zz; }
      if (inner[2] && zz < nz && nb2 > st.nbv[2]) { st.nbv[2] = nb2; st.nbz[2] = z0 + zz; }
    }
  }

  // ---- epilogue: the reference's gates, per pixel
  unsigned nlow = 0;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int i = i0 + p;
    const int members = ((i > 0) + 1 + (i < H - 1)) * ((j > 0) + 1 + (j < W - 1));
    // back from half-range c' to c = 2c' - 1
    float bw = st.bw[p];
    bw = (trusted[p] && bw == -2.f) ? -1.f : 2.f * bw - 1.f;   // window beyond zmax: all -1
    const float bf = 2.f * st.best[p] - 1.f;
    const float nbc = 2.f * st.nbv[p] / (float)members - 1.f;
    bool low = false;
    if (a.mode == kSweepPipeline) {
      if (inner[p]) {
        const float cs = trusted[p] ? bw : bf;
        const int zs = trusted[p] ? st.bwz[p] : st.bestz[p];
        low = (double)cs <= a.alpha;
        const int64_t o = (int64_t)i * a.ldo + j;
        a.dout[o] = (int16_t)(low ? st.nbz[p] : zs);
        a.cout[o] = low ? nbc : cs;
        a.low[o] = (uint8_t)low;
      }
      nlow += (low && i >= a.rows.cnt_lo && i < a.rows.cnt_hi) ? 1u : 0u;
    } else if (inner[p]) {
      const int64_t o = (int64_t)i * W + j;
      a.fz[o] = (int16_t)st.bestz[p];
      a.fc[o] = bf;
      if (a.wz) { a.wz[o] = (int16_t)st.bwz[p]; a.wcst[o] = trusted[p] ? bw : -2.f; }
      a.nz[o] = (int16_t)st.nbz[p];
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

template <int B, int DIR, int ZC, int NR, int NZ, int MINB>
cudaError_t launch3(const SweepArgs& a, cudaStream_t s) {
  constexpr size_t smem = Sweep3Smem<B, ZC, NR>::bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(sweep3_kernel<B, DIR, ZC, NR, NZ, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  constexpr int NROW = 3 * NR;
  // CTA rows stay on the whole-image grid (row bands are bit-identical)
  SweepArgs b = a;
  b.rows.lo = (a.rows.lo / (NROW - 2)) * (NROW - 2);
  dim3 grid((a.W + 29) / 30, (b.rows.hi - b.rows.lo + NROW - 3) / (NROW - 2));
  sweep3_kernel<B, DIR, ZC, NR, NZ, MINB><<<grid, NR * 32, smem, s>>>(b);
  return cudaGetLastError();
}

template <int DIR>
cudaError_t launch3_dir(const SweepArgs& a, cudaStream_t s) {
  switch (a.block) {
    case 3: return launch3<3, DIR, 8, 6, 8, 2>(a, s);
    case 5: return launch3<5, DIR, 8, 6, 8, 2>(a, s);
    case 7: return launch3<7, DIR, 8, 6, 8, 2>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool sweep3_supported(int b) { return b == 3 || b == 5 || b == 7; }

cudaError_t launch_sweep3(const SweepArgs& a, cudaStream_t s) {
  return a.dir > 0 ? launch3_dir<1>(a, s) : launch3_dir<-1>(a, s);
}

}  // namespace mshbm
