// Dense fused ZNCC sweep with the disparities across lanes (level 0, b >= 5).
//
// sweep2 gives every thread a pixel pair and loops over z, so each pixel pays
// its own b x b cross-sum (b^2 + b + 1 FMAs per two pixels).  Here lane l of
// warp w owns one disparity z = zp + 32 w + l for a whole CTA tile of TW x TH
// output pixels and streams the tile's rows top to bottom.  Window sums then
// become separable sliding sums held in registers:
//   V[c]  = sum over the b window rows of L'(r, c) * R'(r, c -+ z)   (per tile column)
//           slid one row per step: + new row product - old row product
//   S[u]  = sum of V over the b columns of cost column u            (sliding)
// about 2 FMAs + 2 adds per (pixel, z) instead of ~b^2 / 2.  L' = L - cL with
// a per-CTA constant cL and R' = R - c (per-level constant, prep_staging);
// each pixel's window is re-centred exactly with its own sum of L':
//   sum (L' - mean L')(R' ) = S - (sum L') * (muR(q) - c).
// Winner-take-all runs across lanes: the half-range cost c' = sat(c/2 + 1/2)
// (as in sweep2) + 1 lies in [1, 2], so its float bits are monotone and fit
// 24 bits; key = (bits - 0x3F800000 + 1) << 5 | (31 - lane) and one REDUX.MAX
// gives the warp's first maximum (smallest z on ties); lane 0 stores it per
// (warp, pixel) and the epilogue merges the warps in z order.  The
// 3x3-summed refinement cost is a sliding 3-row / 3-column sum of c' in
// registers, reduced the same way.  The prior window (trusted pixels) masks
// the keys of lanes outside [c - r, c + r]; untrusted pixels use [0, d].
//
// Lane layouts (s4_plan): one disparity per lane (32 per warp, 128
// registers) or two adjacent ones (64 per warp, 168 registers: LDS.64 /
// LDS.128 of the right samples and normalisers feed both, one REDUX for the
// lane's two keys; same arithmetic per (pixel, z), bit-identical outputs),
// plus, for a search range of four two-disparity warps and <= 32 more, a
// row-split pass in which every warp sweeps a quarter of the tile's rows for
// the same 32 disparities.  DESIGN.md section 6.
//
// Also: R' / (muR - c, 0.5/sigmaR) rows stream through a shared-memory ring
// by 1-D bulk copies (one thread, mbarrier completion); z = d for d a
// multiple of 32 is evaluated once per tile after the sweep (no warp with a
// single useful lane); tiles flagged by the precision guard (kernels.h
// Sweep4Guard) are left to the sweep2 fixup.  DESIGN.md section 6.
//
// Reference semantics: matcher.py:184-193 (full search), 263-320 (prior
// window), 196-233 (3x3-summed refinement); zncc.py:271-287 (cost).
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace mshbm {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTW = 16;          // output columns per CTA
constexpr int kNWMax = 8;        // warps (x 32 disparities) per CTA and pass

__device__ __forceinline__ float fma_sat(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ---- mbarrier + 1-D bulk copies (TMA engine) for the row staging
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Shared-memory layout (runtime TH, warps per pass and key slots).
template <int B, int G = 2, int ZZ = 1>
struct S4Layout {
  static constexpr int NV = kTW + B + 1;        // V columns (TW + 2 cost columns + b - 1)
  static constexpr int NVP = (NV + 3) & ~3;     // row pitch (float4 broadcast loads)
  static constexpr int NC = kTW + 2;            // cost columns (1-pixel halo for 3x3 sums)
  static constexpr int RB = B + 2 * G;          // R ring rows (b + G live + G in flight)
  int th, rwp, mwp, nzw;
  size_t o_bar, o_lt, o_pp, o_rr, o_mr, o_sk, o_rk, o_hs, bytes;
  // ring pitches of the row-split pass (32 disparities, sweep4_kernel run_rows)
  static constexpr int RWS = (NV + 31 + 3 + 3 + 3) & ~3, MWS = (NC + 31 + 1 + 1 + 1) & ~1;
  __host__ __device__ S4Layout(int th_, int nw, int nzw_, bool rows_pass = false)
      : th(th_), nzw(nzw_) {
    // ring rows start 16-byte aligned in global memory: up to 3 (R) / 1 (Mp)
    // extra leading elements, and the copy is rounded up to 16 bytes
    // (ZZ = 2: lanes read whole pairs from the even element at or below
    // their first one, up to 2 more elements either side)
    rwp = (NV + 32 * ZZ * nw - 1 + 3 + 3 + 3 + (ZZ > 1 ? 4 : 0)) & ~3;
    mwp = (NC + 32 * ZZ * nw - 1 + 1 + 1 + 1 + (ZZ > 1 ? 4 : 0)) & ~1;
    size_t o = 0;
    o_bar = o; o += 16;   // the tile's row masks (sel, ref) + the ring's mbarrier
    o_pp = o; o += sizeof(float4) * (th + 2) * (NC / 2);
    // (the row-split pass stages all its rows at once: th + 2 / th + B + 1 short rows)
    const int mre = rows_pass && (th + 2) * MWS > 2 * G * mwp ? (th + 2) * MWS : 2 * G * mwp;
    const int rre = rows_pass && (th + B + 1) * RWS > RB * rwp ? (th + B + 1) * RWS : RB * rwp;
    o_mr = o; o += sizeof(float2) * mre;
    o = (o + 15) & ~(size_t)15;
    o_lt = o; o += sizeof(float) * (th + B + 1) * NVP;
    o_rr = o; o += sizeof(float) * rre;
    o = (o + 15) & ~(size_t)15;
    o_sk = o; o += sizeof(unsigned) * nzw * th * kTW;
    o_rk = o; o += sizeof(unsigned) * nzw * th * kTW;
    o = (o + 15) & ~(size_t)15;
    o_hs = o; o += sizeof(double) * (th + B + 1) * NC;   // prologue only
    bytes = o;
  }
};

// One row step: cost row k (image row y0 - 1 + k).  Xin = 3-sums of row
// k - 1, Xout <- 3-sums of row k, Y = 3-sums of rows k-2 + k-1 on entry and
// rows k-1 + k on exit.  SEL: full-range winner of output row k - 1 (lane 0
// stores the warp's key per pixel into sk); REF: 3x3-summed winner of
// output row k - 2 (into rk).  Rows whose pixels need neither skip the
// reductions (the tile's row masks, see sweep4_kernel).
// TWW: tile columns (kTW); SH: key bits holding the warp-local z.
template <int B, int TWW, int SH>
__device__ __forceinline__ void row_step(
    const int k, const bool SEL, const bool REF, float (&V)[TWW + B + 1], float (&X)[TWW],
    float (&Y)[TWW], const float4* __restrict__ Pp, const float2* __restrict__ mrow,
    const float half, const unsigned laneK, const bool lane0, unsigned* __restrict__ sk,
    unsigned* __restrict__ rk) {
  using SL = S4Layout<B>;
  constexpr int NC = TWW + 2;
  // horizontal window sums S[u] = V[u] + ... + V[u + B - 1]: sliding, as two
  // independent chains (u < NC/2 from S[0], u >= NC/2 from S[NC/2]) over the
  // differences D[u] = V[u + B - 1] - V[u - 1], so the dependent FADD chain is
  // NC/2 deep instead of 2 NC
  float cp[NC];
  {
    constexpr int M = NC / 2;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int c = 0; c < B; ++c) a0 += V[c], a1 += V[M + c];
    cp[0] = a0;
    cp[M] = a1;
#pragma unroll
    for (int u = 1; u < M; ++u) {
      a0 += V[u + B - 1] - V[u - 1];
      a1 += V[M + u + B - 1] - V[M + u - 1];
      cp[u] = a0;
      cp[M + u] = a1;
    }
  }
  // half-range cost c' = sat((S - sumL' * (muR(q) - c)) * kL * 0.5/sigma_R + 1/2);
  // NaN scale (degenerate or out-of-image windows, right centre outside the
  // image) saturates to 0, i.e. c = -1; out-of-image pixels read 0 in 3x3
  // sums.  Lanes with z > d use half = -1e30, so their c' is 0 as well: they
  // never beat a smaller z (ties go to the smaller z) and need no mask.
  const float4* prow = Pp + k * (SL::NC / 2);
#pragma unroll
  for (int u2 = 0; u2 < NC / 2; ++u2) {
    const float4 pp = prow[u2];   // (sumL', kL) of cost columns 2 u2 and 2 u2 + 1
    const float2 m0 = mrow[2 * u2], m1 = mrow[2 * u2 + 1];
    cp[2 * u2] = fma_sat(fmaf(-pp.x, m0.x, cp[2 * u2]) * pp.y, m0.y, half);
    cp[2 * u2 + 1] = fma_sat(fmaf(-pp.z, m1.x, cp[2 * u2 + 1]) * pp.w, m1.y, half);
  }
  // selection (untrusted pixels: the full range [0, d], no window mask):
  // key = (bits(c' + 1) - 0x3F800000 + 1) << SH | (2^SH - 1 - local z),
  // REDUX.MAX = the warp's first maximum
  if (SEL) {
    unsigned* srow = sk + (k - 1) * kTW;
#pragma unroll
    for (int p = 0; p < TWW; ++p) {
      const unsigned key = (__float_as_uint(cp[p + 1] + 1.0f) << SH) + laneK;
      const unsigned r = __reduce_max_sync(kFull, key);
      if (lane0) srow[p] = r;
    }
  }
  // 3x3 sums (horizontal 3-sum of this row + the two rows above in Y) and,
  // for REF rows, their winner; the cost row dies as it is consumed
  unsigned* rrow = rk + (k - 2) * kTW;
  if (REF) {
#pragma unroll
    for (int p = 0; p < TWW; ++p) {
      const float h = (cp[p] + cp[p + 1]) + cp[p + 2];
      const float n = Y[p] + h;
      const unsigned key = (__float_as_uint(fmaf(n, 0.0625f, 1.0f)) << SH) + laneK;
      const unsigned r = __reduce_max_sync(kFull, key);
      if (lane0) rrow[p] = r;
      Y[p] = X[p] + h;
      X[p] = h;
    }
  } else {
#pragma unroll
    for (int p = 0; p < TWW; ++p) {
      const float h = (cp[p] + cp[p + 1]) + cp[p + 2];
      Y[p] = X[p] + h;
      X[p] = h;
    }
  }
}

// Two disparities per lane (ZZ = 2): lane l of warp w owns z0 = zlo + 2 l and
// z0 + 1.  Adjacent disparities read adjacent right samples, so one LDS.64 /
// LDS.128 per lane feeds both (half the shared-memory wavefronts per
// evaluated disparity of the one-disparity layout), the broadcast L' / Pp
// loads are shared, and the lane's two keys are merged before the REDUX.
// Per (pixel, z) the arithmetic and its order are those of row_step, so the
// results are bit-identical.  t-index of the value of column c for
// disparity e of the lane: c + S + (DIR > 0 ? 1 - e : e), S = the parity pad
// of the lane's first element (compile-time, see sweep4_kernel).
template <int DIR>
__device__ __forceinline__ constexpr int zoff(int e) { return DIR > 0 ? 1 - e : e; }

template <int B, int DIR>
__device__ __forceinline__ void row_step2(
    const int k, const bool SEL, const bool REF, float (&V)[2][S4Layout<B>::NV],
    float (&X)[2][kTW], float (&Y)[2][kTW], const float4* __restrict__ Pp,
    const float4* __restrict__ mrow4, const float (&half)[2], const unsigned (&laneK)[2],
    const bool lane0, unsigned* __restrict__ sk, unsigned* __restrict__ rk) {
  using SL = S4Layout<B>;
  constexpr int NC = SL::NC;
  constexpr int sM = DIR > 0 ? 0 : 1;
  constexpr int NT4 = (NC + 1 + sM + 1) / 2;
  float cp[2][NC];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    constexpr int M = NC / 2;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int c = 0; c < B; ++c) a0 += V[e][c], a1 += V[e][M + c];
    cp[e][0] = a0;
    cp[e][M] = a1;
#pragma unroll
    for (int u = 1; u < M; ++u) {
      a0 += V[e][u + B - 1] - V[e][u - 1];
      a1 += V[e][M + u + B - 1] - V[e][M + u - 1];
      cp[e][u] = a0;
      cp[e][M + u] = a1;
    }
  }
  float2 mt[2 * NT4];
#pragma unroll
  for (int i = 0; i < NT4; ++i) {
    const float4 q = mrow4[i];
    mt[2 * i] = make_float2(q.x, q.y);
    mt[2 * i + 1] = make_float2(q.z, q.w);
  }
  const float4* prow = Pp + k * (NC / 2);
#pragma unroll
  for (int u2 = 0; u2 < NC / 2; ++u2) {
    const float4 pp = prow[u2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float2 m0 = mt[2 * u2 + sM + zoff<DIR>(e)], m1 = mt[2 * u2 + 1 + sM + zoff<DIR>(e)];
      cp[e][2 * u2] = fma_sat(fmaf(-pp.x, m0.x, cp[e][2 * u2]) * pp.y, m0.y, half[e]);
      cp[e][2 * u2 + 1] = fma_sat(fmaf(-pp.z, m1.x, cp[e][2 * u2 + 1]) * pp.w, m1.y, half[e]);
    }
  }
  if (SEL) {
    unsigned* srow = sk + (k - 1) * kTW;
#pragma unroll
    for (int p = 0; p < kTW; ++p) {
      const unsigned k0 = (__float_as_uint(cp[0][p + 1] + 1.0f) << 6) + laneK[0];
      const unsigned k1 = (__float_as_uint(cp[1][p + 1] + 1.0f) << 6) + laneK[1];
      const unsigned r = __reduce_max_sync(kFull, max(k0, k1));
      if (lane0) srow[p] = r;
    }
  }
  unsigned* rrow = rk + (k - 2) * kTW;
  if (REF) {
#pragma unroll
    for (int p = 0; p < kTW; ++p) {
      unsigned key[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float h = (cp[e][p] + cp[e][p + 1]) + cp[e][p + 2];
        const float n = Y[e][p] + h;
        key[e] = (__float_as_uint(fmaf(n, 0.0625f, 1.0f)) << 6) + laneK[e];
        Y[e][p] = X[e][p] + h;
        X[e][p] = h;
      }
      const unsigned r = __reduce_max_sync(kFull, max(key[0], key[1]));
      if (lane0) rrow[p] = r;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int p = 0; p < kTW; ++p) {
        const float h = (cp[e][p] + cp[e][p + 1]) + cp[e][p + 2];
        Y[e][p] = X[e][p] + h;
        X[e][p] = h;
      }
  }
}

template <int B, int DIR, int G, int ZZ, int NWM, int REGS>
__global__ void __launch_bounds__(NWM * 32) __maxnreg__(REGS) sweep4_kernel(const SweepArgs a, const int th_,
                                                                               const int ybase) {
  pdl_wait();
  const int th = th_;
  using SL = S4Layout<B, G, ZZ>;
  constexpr int H2 = B / 2, NV = SL::NV, NVP = SL::NVP, NC = SL::NC, RB = SL::RB;
  constexpr int ZW = 32 * ZZ;                 // disparities per warp
  constexpr int SH = ZZ == 1 ? 5 : 6;         // key bits holding the warp-local z
  extern __shared__ float4 smem4[];
  char* smem = reinterpret_cast<char*>(smem4);
  const int nw = blockDim.x >> 5;
  const int d = a.d;
  // d a multiple of 32: the lanes cover z < d and the tail disparity z = d
  // (which would cost a whole warp with one useful lane) is evaluated once
  // per tile after the sweep, as a separable box sum, when that saves a
  // warp slot (the launcher's choice, s4_plan)
  const bool tail = a.s4_tail != 0;
  const int nz = a.s4_ze;    // disparities on lanes: [0, nz)
  // [0, nzm) on the warps' own lanes (ZZ each); the rest, if any, in a
  // row-split pass of all warps (below), one more key slot
  const int nzm = a.s4_zm;
  const int nslot = ((nzm + ZW * nw - 1) / (ZW * nw)) * nw + (nzm < nz ? 1 : 0);
  const SL lay(th, nw, nslot, nzm < nz);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + lay.o_bar) + 1;
  unsigned* sK = reinterpret_cast<unsigned*>(smem + lay.o_sk);
  unsigned* rK = reinterpret_cast<unsigned*>(smem + lay.o_rk);
  float4* Pp = reinterpret_cast<float4*>(smem + lay.o_pp);
  unsigned* masks = reinterpret_cast<unsigned*>(smem + lay.o_bar);
  float2* Mr = reinterpret_cast<float2*>(smem + lay.o_mr);
  float* Lt = reinterpret_cast<float*>(smem + lay.o_lt);
  float* Rr = reinterpret_cast<float*>(smem + lay.o_rr);

  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wp = tid >> 5;
  const int x0 = blockIdx.x * kTW;
  // tile rows on the whole-image grid (ybase: the first one's top row, may be
  // above the image or the stage's rows; a.rows are the rows to compute)
  const int y0 = ybase + blockIdx.y * th;
  const int H = a.H, W = a.W;
  const float qnan = __int_as_float(0x7fc00000);

  // Precision guard: the sliding sums multiply tile-centred values, so their
  // fp32 rounding error relative to the cost scales with the tile's
  // centring amplification (kernels.h Sweep4Guard, evaluated by the L
  // statistics kernel on the statistics branch).  Flagged tiles are left to the per-pixel-centred
  // sweep2 fixup launch (launch_sweep4_fixup), which may run concurrently.
  if (a.tile_flags != nullptr &&
      a.tile_flags[(int64_t)tile_row(y0, th) * a.flags_ld + blockIdx.x] != 0)
    return;   // uniform: the whole CTA leaves
  // ---- which output rows need what.  Pixel states (wc): kWcDone = trusted,
  // not low, finished by prior_select_kernel; kWcLow = trusted and low: only
  // the 3x3-summed refinement; kWcNone (or no prior) = untrusted: full-range
  // selection + refinement.  masks[0] bit o: row o holds an untrusted pixel
  // (SEL), masks[1] bit o: a pixel needing refinement (REF).  Rows outside
  // the stage's rows need nothing.
  if (tid < 2) masks[tid] = 0u;
  __syncthreads();
  for (int t = tid; t < th * kTW; t += nt) {
    const int o = t / kTW, p = t - o * kTW;
    const int y = y0 + o, x = x0 + p;
    if (y < a.rows.lo || y >= a.rows.hi || y >= H || x >= W) continue;
    const int c = a.wc != nullptr ? a.wc[(int64_t)y * a.ldw + x] : kWcNone;
    if (c == kWcNone) atomicOr(&masks[0], 1u << o);
    if (c == kWcNone || c == kWcLow) atomicOr(&masks[1], 1u << o);
  }
  __syncthreads();
  const unsigned selm = masks[0], refm = masks[1];
  if ((selm | refm) == 0u) return;   // uniform: every pixel finished (or none here)
  // ---- prologue: winner slots, left tile L' = L - cL, kL = 1/(b^2 sigma_L)
  // per cost pixel (NaN: degenerate or outside the image); the global loads
  // of both in one phase
  if (tid == 0) mbar_init(bars, 1);
  for (int t = tid; t < nslot * th * kTW; t += nt) sK[t] = 0u, rK[t] = 0u;
  // centring constant: the L sample at the tile centre (the guard in the L
  // statistics kernel uses the same one)
  const double cL = a.Lv(clampi(y0 + th / 2, 0, H - 1), clampi(x0 + kTW / 2, 0, W - 1));
  for (int t = tid; t < (th + B + 1) * NV; t += nt) {
    const int rr = t / NV, c = t - rr * NV;
    const int y = clampi(y0 - 1 - H2 + rr, 0, H - 1), x = clampi(x0 - 1 - H2 + c, 0, W - 1);
    Lt[rr * NVP + c] = (float)(a.Lv(y, x) - cL);
  }
  for (int t = tid; t < (th + 2) * NC; t += nt) {
    const int k = t / NC, u = t - k * NC;
    const int y = y0 - 1 + k, x = x0 - 1 + u;
    float kL = qnan;
    if (y >= 0 && y < H && x >= 0 && x < W) {
      const float is = a.isL[(int64_t)y * a.lds + x];
      if (is > 0.f) kL = is * (1.0f / (float)(B * B));
    }
    reinterpret_cast<float*>(Pp)[2 * t + 1] = kL;
  }
  __syncthreads();
  // cost row k (output row k - 1) is needed by SEL of row k - 1 and REF of
  // rows k - 2, k - 1, k; rows nobody needs skip the cost and reductions
  const unsigned long long needc = ((unsigned long long)selm << 1) |
                                   ((unsigned long long)refm << 2) |
                                   ((unsigned long long)refm << 1) | (unsigned long long)refm;
  // the sweep stops after the last needed cost row (a row band's bottom
  // halo tile needs its first rows only).  It always starts at row 0: the
  // fp32 sliding sums then hold the same values whichever rows a run needs,
  // so row bands stay bit-identical to whole-image runs (a data-dependent
  // start row measured no faster on whole images).
  constexpr int k0 = 0;
  const int kend = 64 - __clzll((long long)needc);
  // per cost pixel: the sum of L' over its window (fp64 sums of the fp32
  // values, so the centring cancels the rounding of L'), separable through
  // per-row horizontal sums, and kL = 1/(b^2 sigma_L)
  double* Hs = reinterpret_cast<double*>(smem + lay.o_hs);
  for (int t = tid; t < (th + B + 1) * NC; t += nt) {
    const int rr = t / NC, u = t - rr * NC;
    const float* lr = Lt + rr * NVP + u;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < B; ++c) s += (double)lr[c];
    Hs[t] = s;
  }
  __syncthreads();
  for (int t = tid; t < (th + 2) * NC; t += nt) {
    const int k = t / NC, u = t - k * NC;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < B; ++r) s += Hs[(k + r) * NC + u];
    reinterpret_cast<float*>(Pp)[2 * t] = (float)s;
  }
  __syncthreads();   // Pp, Lt, the mbarriers

  const float* __restrict__ Rp = a.Rp + a.pc;
  const float2* __restrict__ Mp = a.Mp + a.pc;
  unsigned phase = 0;
  // One pass over the tile's rows for the disparities [zp, zp + ZW * nwp) on
  // the lanes of nwp warps, ZZ per lane; winners into key slot `slot0 + wp`.
  auto run_pass = [&](const int zp, const int nwp, const int slot0, const bool first) {
    const int zlo = zp + ZW * wp;
    const int z = zlo + ZZ * lane;   // the lane's (first) disparity
    // every z of the warp has its right centre outside the image for every
    // cost column of the tile: costs are all -1 there, and lower warps hold
    // smaller z with costs >= -1, so skipping the warp is exact (its key
    // slots stay 0 = no candidate)
    const bool active = wp < nwp && (DIR > 0 ? (zlo <= x0 + kTW) : (zlo <= W - x0));
    const int span = ZW * nwp - 1;
    // image column of ring element 0 (R ring: tile V columns, Mp ring: cost
    // columns), moved down to a 16-byte boundary of the padded row
    int rc0 = DIR > 0 ? (x0 - 1 - H2 - zp - span) : (x0 - 1 - H2 + zp);
    int mc0 = DIR > 0 ? (x0 - 1 - zp - span) : (x0 - 1 + zp);
    const int rmis = (a.pc + rc0) & 3, mmis = (a.pc + mc0) & 1;
    rc0 -= rmis;
    mc0 -= mmis;
    const int rwp = lay.rwp, mwp = lay.mwp;
    const unsigned rbytes = (unsigned)(((NV + span + rmis + 3) & ~3) * sizeof(float));
    const unsigned mbytes = (unsigned)(((NC + span + mmis + 1) & ~1) * sizeof(float2));
    // lane base into the rings: element index of column c for this z.
    // ZZ = 2: the lane's first element (that of z + 1 for DIR > 0) moved down
    // to an even index, so whole pairs load with LDS.64 / LDS.128; the parity
    // pads sR, sM are compile-time constants because x0, zp and the padding
    // column a.pc are even
    constexpr int sR = ZZ == 1 ? 0 : (DIR > 0 ? (H2 & 1) : ((H2 + 1) & 1));
    constexpr int sM = ZZ == 1 ? 0 : (DIR > 0 ? 0 : 1);
    const int lb = (DIR > 0 ? (span - (z - zp)) - (ZZ - 1) : (z - zp)) + rmis - sR;
    const int mb = (DIR > 0 ? (span - (z - zp)) - (ZZ - 1) : (z - zp)) + mmis - sM;
    if (ZZ > 1 && ((lb | mb) & 1)) __trap();

    auto stage_r = [&](int rr, unsigned long long* bar) {
      const int y = clampi(y0 - 1 - H2 + rr, 0, H - 1);
      bulk_g2s(Rr + (rr % RB) * rwp, Rp + ((int64_t)y * a.ldp + rc0), rbytes, bar);
    };
    auto stage_m = [&](int k, unsigned long long* bar) {
      const int y = clampi(y0 - 1 + k, 0, H - 1);
      bulk_g2s(Mr + (k % (2 * G)) * mwp, Mp + ((int64_t)y * a.ldp + mc0), mbytes, bar);
    };
    if (!first) __syncthreads();   // previous pass done with the rings

    if (tid == 0) {
      fence_proxy_async();
      const int nr0 = min(B + G, th + B + 1 - k0), nm0 = min(G, th + 2 - k0);
      mbar_expect_tx(bars, nr0 * rbytes + nm0 * mbytes);
      for (int rr = k0; rr < k0 + nr0; ++rr) stage_r(rr, bars);
      for (int k = k0; k < k0 + nm0; ++k) stage_m(k, bars);
    }
    mbar_wait(bars, phase & 1u);
    phase ^= 1u;

    float V[ZZ][NV];
    constexpr int NT2 = (NV + 1 + sR + 1) / 2;   // ZZ = 2: float2 loads per ring row
    // ring row -> the lane's NV + 1 (+ pad) consecutive samples
    auto load_r = [&](const float* rowp, float (&t)[2 * NT2]) {
      const float2* rp = reinterpret_cast<const float2*>(rowp + lb);
#pragma unroll
      for (int i = 0; i < NT2; ++i) {
        const float2 v = rp[i];
        t[2 * i] = v.x;
        t[2 * i + 1] = v.y;
      }
    };
    // V[.][c] += sign * L'(row, c) * R'(ring row, c -+ z) over the warp's columns
    auto accum = [&](int lrow, int ring_row) {
      const float4* lr = reinterpret_cast<const float4*>(Lt + lrow * NVP);
      if constexpr (ZZ == 1) {
        const float* rrow = Rr + ring_row * rwp + lb;
#pragma unroll
        for (int c4 = 0; c4 < NVP / 4; ++c4) {
          const float4 l4 = lr[c4];
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * c4 + e;
            if (c < NV) V[0][c] = fmaf(lv[e], rrow[c], V[0][c]);
          }
        }
      } else {
        float t[2 * NT2];
        load_r(Rr + ring_row * rwp, t);
#pragma unroll
        for (int c4 = 0; c4 < NVP / 4; ++c4) {
          const float4 l4 = lr[c4];
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * c4 + e;
            if (c < NV) {
              V[0][c] = fmaf(lv[e], t[c + sR + zoff<DIR>(0)], V[0][c]);
              V[1][c] = fmaf(lv[e], t[c + sR + zoff<DIR>(1)], V[1][c]);
            }
          }
        }
      }
    };
    if (active) {
#pragma unroll
      for (int e = 0; e < ZZ; ++e)
#pragma unroll
        for (int c = 0; c < NV; ++c) V[e][c] = 0.f;
#pragma unroll
      for (int r = 0; r < B; ++r) accum(k0 + r, (k0 + r) % RB);
    }
    const bool lane0 = lane == 0;
    unsigned laneK[ZZ];
    float half[ZZ];
#pragma unroll
    for (int e = 0; e < ZZ; ++e) {
      laneK[e] = (unsigned)(ZW - 1 - (ZZ * lane + e)) + (1u << SH) - (0x3F800000u << SH);
      half[e] = z + e < nz ? 0.5f : -1.0e30f;
    }
    unsigned* sk = sK + (slot0 + wp) * th * kTW;
    unsigned* rk = rK + (slot0 + wp) * th * kTW;
    float X[ZZ][kTW], Y[ZZ][kTW];
#pragma unroll
    for (int e = 0; e < ZZ; ++e)
#pragma unroll
      for (int p = 0; p < kTW; ++p) X[e][p] = 0.f, Y[e][p] = 0.f;

    // Rows are consumed in groups of G steps: one mbarrier wait and one CTA
    // barrier per group; the ring holds the group's b + G R rows and G Mp
    // rows plus the next group's, prefetched by one thread with bulk copies.
    // One copy of the step body (instruction cache): the SEL / REF
    // reductions are warp-uniform branches on the tile's row masks.
    auto step = [&](int k) {
      if (active) {
        if ((needc >> k) & 1ull) {
          const bool sl = k >= 1 && ((selm >> (k - 1)) & 1u);
          const bool rf = k >= 2 && ((refm >> (k - 2)) & 1u);
          const float2* mrow = Mr + (k % (2 * G)) * mwp + mb;
          if constexpr (ZZ == 1)
            row_step<B, kTW, SH>(k, sl, rf, V[0], X[0], Y[0], Pp, mrow, half[0],
                                  laneK[0], lane0, sk, rk);
          else
            row_step2<B, DIR>(k, sl, rf, V, X, Y, Pp, reinterpret_cast<const float4*>(mrow), half,
                              laneK, lane0, sk, rk);
        }
        // slide V down one row: + row k + B, - row k
        if (k <= th) {
          const float4* lin = reinterpret_cast<const float4*>(Lt + (k + B) * NVP);
          const float4* lout = reinterpret_cast<const float4*>(Lt + k * NVP);
          if constexpr (ZZ == 1) {
            const float* rin = Rr + ((k + B) % RB) * rwp + lb;
            const float* rout = Rr + (k % RB) * rwp + lb;
#pragma unroll
            for (int c4 = 0; c4 < NVP / 4; ++c4) {
              const float4 i4 = lin[c4], o4 = lout[c4];
              const float iv[4] = {i4.x, i4.y, i4.z, i4.w}, ov[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = 4 * c4 + e;
                if (c < NV) V[0][c] = fmaf(iv[e], rin[c], fmaf(-ov[e], rout[c], V[0][c]));
              }
            }
          } else {
            float tin[2 * NT2], tout[2 * NT2];
            load_r(Rr + ((k + B) % RB) * rwp, tin);
            load_r(Rr + (k % RB) * rwp, tout);
#pragma unroll
            for (int c4 = 0; c4 < NVP / 4; ++c4) {
              const float4 i4 = lin[c4], o4 = lout[c4];
              const float iv[4] = {i4.x, i4.y, i4.z, i4.w}, ov[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = 4 * c4 + e;
                if (c < NV) {
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const int j = c + sR + zoff<DIR>(q);
                    V[q][c] = fmaf(iv[e], tin[j], fmaf(-ov[e], tout[j], V[q][c]));
                  }
                }
              }
            }
          }
        }
      }
    };
#pragma unroll 1
    for (int k = k0; k < kend; k += G) {
      if (k > k0) {
        mbar_wait(bars, phase & 1u);
        phase ^= 1u;
        __syncthreads();   // every warp done with the previous group (its slots are reused)
      }
      if (tid == 0 && k + G < kend) {
        fence_proxy_async();
        const int r0 = k + B + G, r1 = min(k + B + 2 * G, th + B + 1);
        const int m0 = k + G, m1 = min(k + 2 * G, th + 2);
        mbar_expect_tx(bars, max(r1 - r0, 0) * rbytes + (m1 - m0) * mbytes);
        for (int rr = r0; rr < r1; ++rr) stage_r(rr, bars);
        for (int km = m0; km < m1; ++km) stage_m(km, bars);
      }
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        if (k + g < kend) step(k + g);
      }
    }
  };
  // the warps' own disparities: [0, nzm), ZZ per lane
  int pass = 0;
  for (int zp = 0; zp < nzm; zp += ZW * nw, ++pass)
    run_pass(zp, min(nw, (nzm - 1 - zp) / ZW + 1), pass * nw, pass == 0);
  // The remaining <= 32 disparities [nzm, nz) (two-disparity kernels with
  // 4-warp CTAs): instead of a fifth warp, which would leave the SM's four
  // schedulers with 3, 3, 2, 2 warps, every warp holds the same 32
  // disparities, one per lane, and sweeps a quarter of the tile's rows (its
  // output rows + the 2 more cost rows their 3x3 sums read) with sliding
  // sums started at its own first row.  The rows of so narrow a range are
  // short, so all of them are staged at once: no barrier inside the pass.
  if constexpr (ZZ == 2) {
    if (nzm < nz) {
      constexpr int RWS = SL::RWS, MWS = SL::MWS, span = 31;
      const int zp = nzm, z = zp + lane;
      const bool active = DIR > 0 ? (zp <= x0 + kTW) : (zp <= W - x0);
      int rc0 = DIR > 0 ? (x0 - 1 - H2 - zp - span) : (x0 - 1 - H2 + zp);
      int mc0 = DIR > 0 ? (x0 - 1 - zp - span) : (x0 - 1 + zp);
      const int rmis = (a.pc + rc0) & 3, mmis = (a.pc + mc0) & 1;
      rc0 -= rmis;
      mc0 -= mmis;
      const unsigned rbytes = (unsigned)(((NV + span + rmis + 3) & ~3) * sizeof(float));
      const unsigned mbytes = (unsigned)(((NC + span + mmis + 1) & ~1) * sizeof(float2));
      const int lb = (DIR > 0 ? span - lane : lane) + rmis;
      const int mb = (DIR > 0 ? span - lane : lane) + mmis;
      __syncthreads();   // the warps' own passes are done with the rings
      const int nrr = min(kend + B, th + B + 1), nmr = min(kend, th + 2);
      if (tid == 0) {
        fence_proxy_async();
        mbar_expect_tx(bars, nrr * rbytes + nmr * mbytes);
        for (int rr = 0; rr < nrr; ++rr)
          bulk_g2s(Rr + rr * RWS, Rp + ((int64_t)clampi(y0 - 1 - H2 + rr, 0, H - 1) * a.ldp + rc0),
                   rbytes, bars);
        for (int k = 0; k < nmr; ++k)
          bulk_g2s(Mr + k * MWS, Mp + ((int64_t)clampi(y0 - 1 + k, 0, H - 1) * a.ldp + mc0), mbytes,
                   bars);
      }
      mbar_wait(bars, phase & 1u);
      phase ^= 1u;
      const int rows_w = (th + nw - 1) / nw;            // output rows per warp
      const int klo = rows_w * wp, khi = min(klo + rows_w + 2, kend);
      if (active && klo < khi) {
        float V[NV], X[kTW], Y[kTW];
#pragma unroll
        for (int c = 0; c < NV; ++c) V[c] = 0.f;
#pragma unroll
        for (int p = 0; p < kTW; ++p) X[p] = 0.f, Y[p] = 0.f;
        // V[c] += L'(lrow, c) * R'(lrow, c -+ z)
        auto accum = [&](int lrow) {
          const float4* lr = reinterpret_cast<const float4*>(Lt + lrow * NVP);
          const float* rrow = Rr + lrow * RWS + lb;
#pragma unroll
          for (int c4 = 0; c4 < NVP / 4; ++c4) {
            const float4 l4 = lr[c4];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 4 * c4 + e;
              if (c < NV) V[c] = fmaf(lv[e], rrow[c], V[c]);
            }
          }
        };
#pragma unroll 1
        for (int r = 0; r < B; ++r) accum(klo + r);
        const unsigned laneK = (unsigned)(ZW - 1 - lane) + (1u << SH) - (0x3F800000u << SH);
        const float half = z < nz ? 0.5f : -1.0e30f;
        unsigned* sk = sK + (nslot - 1) * th * kTW;
        unsigned* rk = rK + (nslot - 1) * th * kTW;
#pragma unroll 1
        for (int k = klo; k < khi; ++k) {
          if ((needc >> k) & 1ull) {
            // this warp's output rows only: [klo, klo + rows_w)
            const bool sl = k >= klo + 1 && k <= klo + rows_w && ((selm >> (k - 1)) & 1u);
            const bool rf = k >= klo + 2 && ((refm >> (k - 2)) & 1u);
            row_step<B, kTW, SH>(k, sl, rf, V, X, Y, Pp, Mr + k * MWS + mb, half, laneK, lane == 0,
                                 sk, rk);
          }
          if (k + 1 < khi) {   // slide V down one row: + row k + B, - row k
            const float4* lin = reinterpret_cast<const float4*>(Lt + (k + B) * NVP);
            const float4* lout = reinterpret_cast<const float4*>(Lt + k * NVP);
            const float* rin = Rr + (k + B) * RWS + lb;
            const float* rout = Rr + k * RWS + lb;
#pragma unroll
            for (int c4 = 0; c4 < NVP / 4; ++c4) {
              const float4 i4 = lin[c4], o4 = lout[c4];
              const float iv[4] = {i4.x, i4.y, i4.z, i4.w}, ov[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = 4 * c4 + e;
                if (c < NV) V[c] = fmaf(iv[e], rin[c], fmaf(-ov[e], rout[c], V[c]));
              }
            }
          }
        }
      }
    }
  }
  __syncthreads();

  // ---- tail disparity z = d: half-range costs c'(d) of every cost pixel
  // (TH + 2 rows x TW + 2 columns) into Ct, from row sums Ht of L' x R'
  float* Ct = reinterpret_cast<float*>(smem + lay.o_hs);
  float* Ht = Ct + (th + 2) * NC;
  if (tail) {
    const int qd = DIR > 0 ? -d : d;   // right column offset of z = d
    for (int t = tid; t < (th + B + 1) * NC; t += nt) {
      const int rr = t / NC, u = t - rr * NC;
      const int y = clampi(y0 - 1 - H2 + rr, 0, H - 1);
      const float* rrow = Rp + ((int64_t)y * a.ldp + (x0 - 1 - H2 + u + qd));
      const float* lr = Lt + rr * NVP + u;
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < B; ++c) acc = fmaf(lr[c], __ldg(rrow + c), acc);
      Ht[t] = acc;
    }
    __syncthreads();
    for (int t = tid; t < (th + 2) * NC; t += nt) {
      const int k = t / NC, u = t - k * NC;
      float S = 0.f;
#pragma unroll
      for (int r = 0; r < B; ++r) S += Ht[(k + r) * NC + u];
      const float* pf = reinterpret_cast<const float*>(Pp) + 2 * t;
      const int yc = clampi(y0 - 1 + k, 0, H - 1);
      const float2 m = Mp[(int64_t)yc * a.ldp + (x0 - 1 + u + qd)];
      Ct[t] = fma_sat(fmaf(-pf[0], m.x, S) * pf[1], m.y, 0.5f);
    }
    __syncthreads();
  }

  // ---- epilogue: merge the warps' winners (lower warp = smaller z first on
  // ties), then the reference's gates, per output pixel
  unsigned nlow = 0;
  for (int t = tid; t < th * kTW; t += nt) {
    const int o = t / kTW, p = t - o * kTW;
    const int i = y0 + o, j = x0 + p;
    if (i >= H || j >= W || i < a.rows.lo || i >= a.rows.hi) continue;
    const int wcp = a.wc != nullptr ? a.wc[(int64_t)i * a.ldw + j] : kWcNone;
    if (wcp != kWcNone && wcp != kWcLow) continue;   // finished by prior_select_kernel
    const bool sel = wcp == kWcNone;   // untrusted: full-range selection first
    unsigned bs = 0u, br = 0u;
    int zs = -1, nbz = 0;
    for (int w = 0; w < nslot; ++w) {
      const unsigned ks = sK[w * th * kTW + t], kr = rK[w * th * kTW + t];
      if ((ks >> SH) > (bs >> SH)) bs = ks, zs = ZW * w + ZW - 1 - (int)(ks & (unsigned)(ZW - 1));
      if ((kr >> SH) > (br >> SH)) br = kr, nbz = ZW * w + ZW - 1 - (int)(kr & (unsigned)(ZW - 1));
    }
    if (zs < 0) {
      // no candidate on an active warp: every right centre is outside the
      // image, all -1 (value 1), smallest z
      bs = 1u << SH;
      zs = 0;
    }
    if (tail) {   // z = d last: it wins only if strictly better
      const float* ct = Ct + o * NC + p;
      const unsigned vd = __float_as_uint(ct[NC + 1] + 1.0f) - 0x3F800000u + 1u;
      if (vd > (bs >> SH)) bs = vd << SH, zs = d;
      const float nsum = (((ct[0] + ct[1]) + ct[2]) + ((ct[NC] + ct[NC + 1]) + ct[NC + 2])) +
                         ((ct[2 * NC] + ct[2 * NC + 1]) + ct[2 * NC + 2]);
      const unsigned vn = __float_as_uint(fmaf(nsum, 0.0625f, 1.0f)) - 0x3F800000u + 1u;
      if (vn > (br >> SH)) br = vn << SH, nbz = d;
    }
    const float cs = 2.f * __uint_as_float((bs >> SH) - 1u + 0x3F800000u) - 3.f;  // c = 2 c' - 1
    const float n1 = __uint_as_float((br >> SH) - 1u + 0x3F800000u);
    const float nsum = (n1 - 1.0f) * 16.0f;
    const int members = ((i > 0) + 1 + (i < H - 1)) * ((j > 0) + 1 + (j < W - 1));
    const float nbc = 2.f * nsum / (float)members - 1.f;
    // trusted low pixels were counted by prior_select_kernel
    const bool low = !sel || (double)cs <= a.alpha;
    const int64_t off = (int64_t)i * a.ldo + j;
    a.dout[off] = (int16_t)(low ? nbz : zs);
    a.cout[off] = low ? nbc : cs;
    a.low[off] = (uint8_t)low;
    nlow += (sel && low && i >= a.rows.cnt_lo && i < a.rows.cnt_hi) ? 1u : 0u;
  }
  const int slot[1] = {kCntRefined};
  const unsigned long long val[1] = {nlow};
  const bool mx[1] = {false};
  block_accumulate<1>(a.counters, slot, val, mx);
}

// Trusted-window selection of a sweep4 level (matcher.py:263-320, prior
// window +-r), before the dense sweep.  For every trusted pixel the <= 2r+1
// candidates [c - r, c + r] & [0, d] are scored directly, ascending z with a
// strict >, so ties keep the smallest z.  Non-low pixels get their final
// outputs here and are marked kWcDone (the sweep skips them); low pixels are
// marked kWcLow and counted (the sweep computes only their 3x3-summed
// refinement, matcher.py:196-233); untrusted pixels keep kWcNone.  Tiles the
// precision guard flagged are left whole to the sweep2 fixup.
//
// Centring: with L'' = fl32(L - m) for any constant m near the window's mean
// (one rounding per value) and R' = fl32(R - c) (staging), the centred
// cross sum of a window W is
//   sum_W L'' R' - (sum_W L'') (muR(q) - c)
// (sum_W R' = b^2 (muR(q) - c)), whichever m was subtracted; sum_W L'' is
// accumulated in fp64, so it cancels the rounding of the centring exactly.
// The 2x nearest-neighbour prior gives the pixels (2m, j) and (2m+1, j) the
// same window centre, so one thread scores both: their windows share b - 1
// rows, L'' is centred once (on the upper pixel's mean) and every shared row
// feeds both, (b + 1) x b x (2r + 1) FMAs for two pixels instead of
// 2 x b^2 x (2r + 1).  A 32 x 16-pixel tile of L is staged in shared memory;
// the right span of one window row sits in registers.
// one window row r (image row y) of one window centre: acc[zi] += sum over
// the row of L''(cc) R'(cc -+ (lo + zi)), rs += sum of the row's L'' (fp64)
template <int B, int DIR, int MAXW, typename LT>
__device__ __forceinline__ void psel_row(const SweepArgs& a, const LT* lrow,
                                         const float* __restrict__ Rp, int y, float m,
                                         float (&acc)[MAXW], double& rs) {
  constexpr int NRV = B + MAXW - 1;
  const float* __restrict__ rrow = Rp + (int64_t)clampi(y, 0, a.H - 1) * a.ldp;
  float rv[NRV], l[B];
#pragma unroll
  for (int e = 0; e < NRV; ++e) rv[e] = __ldg(rrow + e);
#pragma unroll
  for (int cc = 0; cc < B; ++cc) {
    if constexpr (std::is_same<LT, float>::value) l[cc] = lrow[cc] - m;
    else l[cc] = (float)(lrow[cc] - (double)m);
  }
#pragma unroll
  for (int cc = 0; cc < B; ++cc) {
    rs += (double)l[cc];
#pragma unroll
    for (int zi = 0; zi < MAXW; ++zi)
      acc[zi] = fmaf(l[cc], rv[DIR > 0 ? cc + MAXW - 1 - zi : cc + zi], acc[zi]);
  }
}

template <int B, int DIR, int MAXW, bool F32>
__global__ void __launch_bounds__(256, 4) prior_select_kernel(const SweepArgs a, const int th) {
  pdl_wait();
  constexpr int H2 = B / 2;
  constexpr int TR = 16 + B - 1, TC = 32 + B - 1;   // left tile (replicate-clamped)
  using LT = typename std::conditional<F32, float, double>::type;
  __shared__ LT Ls[TR][TC];
  const int x0 = blockIdx.x * 32, y0 = (a.rows.lo & ~1) + blockIdx.y * 16;
  const int j = x0 + threadIdx.x, iA = y0 + 2 * threadIdx.y;
  const int H = a.H, W = a.W;
  for (int t = threadIdx.x + 32 * threadIdx.y; t < TR * TC; t += 256) {
    const int rr = t / TC, cc = t - rr * TC;
    const int y = clampi(y0 - H2 + rr, 0, H - 1), x = clampi(x0 - H2 + cc, 0, W - 1);
    if constexpr (F32) Ls[rr][cc] = a.L32[(int64_t)y * a.ld32 + x];
    else Ls[rr][cc] = a.L[(int64_t)y * a.ld + x];
  }
  __syncthreads();
  int* wc = const_cast<int*>(a.wc);
  unsigned nlow = 0;
  // trusted window centre of pixel (i, j) in this stage's rows, else kWcNone
  auto centre = [&](int i) -> int {
    if (i < a.rows.lo || i >= a.rows.hi || i >= H || j >= W) return kWcNone;
    const int c = wc[(int64_t)i * a.ldw + j];
    if (c <= kWcLow) return kWcNone;
    if (a.tile_flags != nullptr &&
        a.tile_flags[(int64_t)tile_row(i, th) * a.flags_ld + (j >> 4)] != 0)
      return kWcNone;
    return c;
  };
  const int cA = centre(iA), cB = centre(iA + 1);
  // score pixel i's window [lo, lo + nw) from its cross sums S and the fp64
  // sum of its L'' values; write / mark it
  auto finish = [&](int i, int lo, int nw, const float (&S)[MAXW], double sumL) {
    const float is = a.isL[(int64_t)i * a.lds + j];
    const float kL = is > 0.f ? is * (1.0f / (float)(B * B)) : __int_as_float(0x7fc00000);
    const float sl = (float)sumL;
    const float2* __restrict__ Mrow = a.Mp + a.pc + (int64_t)i * a.ldp;
    float best = -1.f;
    int bz = lo;
#pragma unroll
    for (int zi = 0; zi < MAXW; ++zi) {
      if (zi < nw) {
        const int z = lo + zi;
        const float2 mm = Mrow[DIR > 0 ? j - z : j + z];
        const float cp = fma_sat(fmaf(-sl, mm.x, S[zi]) * kL, mm.y, 0.5f);
        if (cp > best) best = cp, bz = z;
      }
    }
    const float cs = 2.f * best - 1.f;   // c = 2 c' - 1
    const bool low = (double)cs <= a.alpha;
    const int64_t o = (int64_t)i * a.ldo + j;
    if (low) {
      wc[(int64_t)i * a.ldw + j] = kWcLow;
      nlow += (i >= a.rows.cnt_lo && i < a.rows.cnt_hi) ? 1u : 0u;
    } else {
      a.dout[o] = (int16_t)bz;
      a.cout[o] = cs;
      a.low[o] = 0;
      wc[(int64_t)i * a.ldw + j] = kWcDone;
    }
  };
  // one pass over the rows of one window centre c: rows iA - H2 .. iA + H2
  // (+ one more for the pair), centred on pixel i0's fp32 mean
  auto score = [&](int c, int i0, bool pair, bool fin0, bool fin1) {
    const int lo = max(c - a.radius, 0), hi = min(c + a.radius, a.d);
    const int nw = hi - lo + 1;   // >= 1: trusted windows meet [0, d] (prior)
    const float m = a.muL[(int64_t)i0 * a.lds + j];
    float S0[MAXW], P[MAXW], S1[MAXW];
#pragma unroll
    for (int zi = 0; zi < MAXW; ++zi) S0[zi] = 0.f, P[zi] = 0.f, S1[zi] = 0.f;
    double sum0 = 0.0, sP = 0.0, sum1 = 0.0;
    // first staged right column of the window rows: z = lo + zi reads column
    // j - H2 + cc - z (middlebury) or j - H2 + cc + z (paper)
    const int base = DIR > 0 ? (j - H2 - (lo + MAXW - 1)) : (j - H2 + lo);
    const float* Rp = a.Rp + a.pc + base;
    const LT* l0 = &Ls[i0 - y0][threadIdx.x];
    // row 0: pixel i0 only; rows 1 .. b-1: shared; row b: pixel i0 + 1 only
    psel_row<B, DIR, MAXW, LT>(a, l0, Rp, i0 - H2, m, S0, sum0);
#pragma unroll 1
    for (int r = 1; r < B; ++r) psel_row<B, DIR, MAXW, LT>(a, l0 + r * TC, Rp, i0 - H2 + r, m, P, sP);
    if (pair) psel_row<B, DIR, MAXW, LT>(a, l0 + B * TC, Rp, i0 - H2 + B, m, S1, sum1);
    float SA[MAXW];
#pragma unroll
    for (int zi = 0; zi < MAXW; ++zi) SA[zi] = S0[zi] + P[zi];
    if (fin0) finish(i0, lo, nw, SA, sum0 + sP);
    if (pair && fin1) {
#pragma unroll
      for (int zi = 0; zi < MAXW; ++zi) SA[zi] = P[zi] + S1[zi];
      finish(i0 + 1, lo, nw, SA, sP + sum1);
    }
  };
  // every lane with a trusted pixel runs the same pair pass (no divergent
  // single-pixel paths); the 2x NN prior gives both pixels the same centre,
  // so a second pass is only needed for centres that differ
  if (cA != kWcNone || cB != kWcNone) {
    const int c = cA != kWcNone ? cA : cB;
    score(c, iA, true, cA != kWcNone, cB != kWcNone && cB == c);
    if (cB != kWcNone && cB != c) score(cB, iA + 1, false, true, false);
  }
  const int slot[1] = {kCntRefined};
  const unsigned long long val[1] = {nlow};
  const bool mx[1] = {false};
  block_accumulate<1>(a.counters, slot, val, mx);
}

}  // namespace

int g_th = -1;
int sweep4_th() {
  if (g_th < 0) {
    const char* v = getenv("MSHBM_SWEEP4_TH");
    g_th = v ? atoi(v) : 32;
    // <= 32: the band plans size their statistics halos for 32-row tiles
    if (g_th < 2 || (g_th & 1) || g_th > 32) g_th = 32;
  }
  return g_th;
}

namespace {

template <int B, int DIR, bool F32>
cudaError_t launch_prior_select(const SweepArgs& a, int th, dim3 pg, cudaStream_t s) {
  const dim3 blk(32, 8);
  switch (a.radius) {
    case 0:
    case 1: return launch_pdl(prior_select_kernel<B, DIR, 3, F32>, pg, blk, 0, s, a, th);
    case 2: return launch_pdl(prior_select_kernel<B, DIR, 5, F32>, pg, blk, 0, s, a, th);
    case 3: return launch_pdl(prior_select_kernel<B, DIR, 7, F32>, pg, blk, 0, s, a, th);
    default: return launch_pdl(prior_select_kernel<B, DIR, 15, F32>, pg, blk, 0, s, a, th);
  }
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// CTA shape for `nz` disparities on the lanes, `zw` per warp, <= nwmax warps
// per CTA: passes x warps (the kernel's key slots)
struct S4Shape {
  int passes, nw;
  int slots() const { return passes * nw; }
};
S4Shape s4_shape(int nz, int zw, int nwmax) {
  const int nzw = (nz + zw - 1) / zw;
  S4Shape r;
  r.passes = (nzw + nwmax - 1) / nwmax;
  r.nw = (nzw + r.passes - 1) / r.passes;
  return r;
}

// NWM warps per CTA at most, REGS registers per thread at most
template <int B, int DIR, int G, int ZZ, int NWM, int REGS>
cudaError_t launch4(const SweepArgs& a, S4Shape sh, int slots, cudaStream_t s) {
  const int th = sweep4_th();
  const S4Layout<B, G, ZZ> lay(th, sh.nw, slots, a.s4_zm < a.s4_ze);
  static SmemAttr attr;
  if (cudaError_t e = attr.ensure(sweep4_kernel<B, DIR, G, ZZ, NWM, REGS>, lay.bytes); e != cudaSuccess)
    return e;
  // CTA rows on the whole-image grid (row bands bit-identical to whole runs)
  const int ybase = tile_row(a.rows.lo, th) * th - kTileOff;
  dim3 grid((a.W + kTW - 1) / kTW, (a.rows.hi - ybase + th - 1) / th);
  return launch_pdl(sweep4_kernel<B, DIR, G, ZZ, NWM, REGS>, grid, dim3(32 * sh.nw), lay.bytes, s, a, th,
                    ybase);
}

}  // namespace

bool sweep4_supported(const SweepArgs& a, bool force) {
  // small levels (C1's 450 x 375) leave most SMs idle with one-disparity-
  // per-lane tiles; sweep2's pixel-pair threads are faster there (measured).
  // force (MSHBM_SWEEP4=2) drops the size rule: parity tests on small images
  return (force || (int64_t)a.H * a.W >= 400000) && a.mode == kSweepPipeline &&
         a.muL != nullptr && a.isL != nullptr && a.tile_flags != nullptr &&
         (a.block == 5 || a.block == 7 || a.block == 9 || a.block == 11) &&
         a.d >= 1 &&
         a.d <= 4095 && a.radius <= 7;   // prior_select_kernel: windows of <= 15
}

namespace {

int g_zz = -1;
int sweep4_zz() {
  if (g_zz < 0) {
    g_zz = env_int("MSHBM_SWEEP4_ZZ", 0);   // disparities per lane (1 or 2; 0: by shape)
    if (g_zz != 1 && g_zz != 2) g_zz = 0;
  }
  return g_zz;
}

// How launch_sweep4 lays the search range [0, d] out.  zz: disparities per
// lane.  Two per lane (64 per warp, 168 registers: 3 warps per scheduler)
// halve the shared-memory wavefronts per evaluated disparity and win when
// the CTAs fill the SM's four schedulers evenly (2, 3 or 4 warps, <= 4 so
// that 3 CTAs are resident) without idle lanes beyond what one disparity
// per lane (32 per warp, 128 registers, <= 8 warps) would leave; measured:
// C5 (d = 512) 41.7 -> 34.3 ms, C3 (d = 288, 4.5 warps of 64) no gain.
// tail: z = d is evaluated once per tile after the sweep instead of on a
// lane when it would be a warp's only disparity (d a multiple of the warp's
// range).
// Two per lane need even ring bases: padded rows (a.pc, a.ldp) in multiples
// of 4 elements (prep_staging lays them out so).
struct S4Plan {
  int zz, tail, ze, zm;   // zm: end of the warps' own disparities (== ze: no split pass)
  S4Shape shape;
  int slots() const { return shape.slots() + (zm < ze ? 1 : 0); }
};
S4Plan s4_plan(const SweepArgs& a) {
  auto plan = [&](int zz, int nwmax) {
    const int zw = 32 * zz;
    S4Plan p;
    p.zz = zz;
    p.tail = a.d % zw == 0;   // z = d would take a warp of its own through a pass
    p.zm = p.ze = p.tail ? a.d : a.d + 1;
    p.shape = s4_shape(p.ze, zw, nwmax);
    return p;
  };
  static const int nw1 = max(1, min(8, env_int("MSHBM_SWEEP4_NW", 8)));
  static const int nw2 = max(1, min(4, env_int("MSHBM_SWEEP4_NW", 4)));
  const S4Plan p1 = plan(1, nw1), p2 = plan(2, nw2);
  const bool even = (a.pc & 3) == 0 && (a.ldp & 3) == 0;
  const int zz = sweep4_zz();   // 0: choose, 1 / 2: forced
  if (!even || zz == 1) return p1;
  // Four two-disparity warps and <= 32 disparities more (C3: d = 288): the
  // rest goes to a row-split pass of the same CTA (sweep4_kernel) instead of
  // a fifth warp, which would leave the SM's schedulers with 3, 3, 2, 2
  // warps.  C3 level 0: 2.20 -> 1.84 ms.  (Two full warps + a row-split
  // pass, C2's d = 144: slower than one per lane, 0.41 vs 0.35 ms: the
  // staged rows leave room for 4 CTAs = 8 warps per SM only.)
  static const int split = env_int("MSHBM_SWEEP4_SPLIT", 1);
  if (split && p1.ze > 256 && p1.ze <= 288 && nw2 == 4) {
    S4Plan m = p1;   // the one-disparity tail rule: the split pass holds 32 per warp
    m.zz = 2;
    m.zm = 256;
    m.shape = S4Shape{1, 4};
    return m;
  }
  const bool pick2 = zz == 2 || (p2.shape.nw >= 2 && 64 * p2.shape.slots() <= 32 * p1.shape.slots());
  return pick2 ? p2 : p1;
}

template <int B, int DIR>
cudaError_t launch4_d(const SweepArgs& a0, cudaStream_t s) {
  const int th = sweep4_th();
  if (a0.wc != nullptr) {   // trusted windows first (prior_select_kernel)
    dim3 pg((a0.W + 31) / 32, (a0.rows.hi - (a0.rows.lo & ~1) + 15) / 16);
    cudaError_t e = a0.L32 != nullptr ? launch_prior_select<B, DIR, true>(a0, th, pg, s)
                                       : launch_prior_select<B, DIR, false>(a0, th, pg, s);
    if (e != cudaSuccess) return e;
  }
  const S4Plan p = s4_plan(a0);
  SweepArgs a = a0;
  a.s4_tail = p.tail;
  a.s4_ze = p.ze;
  a.s4_zm = p.zm;
  if (p.zz == 2) return launch4<B, DIR, 2, 2, 4, 168>(a, p.shape, p.slots(), s);
  return launch4<B, DIR, 2, 1, 8, 128>(a, p.shape, p.slots(), s);
}

template <int B>
cudaError_t launch4_b(const SweepArgs& a, cudaStream_t s) {
  return a.dir > 0 ? launch4_d<B, 1>(a, s) : launch4_d<B, -1>(a, s);
}

}  // namespace

cudaError_t launch_sweep4(const SweepArgs& a, cudaStream_t s) {
  switch (a.block) {
    case 5: return launch4_b<5>(a, s);
    case 7: return launch4_b<7>(a, s);
    case 9: return launch4_b<9>(a, s);
    case 11: return launch4_b<11>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mshbm
