// libmshbm: context, per-shape execution plans (CUDA-graph captured), level
// orchestration of run_pipeline, CostEngine handles and the C ABI declared
// in include/mshbm.h.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mshbm.h"
#include "common.cuh"
#include "kernels.h"

using namespace mshbm;

namespace {

thread_local std::string g_err;

}  // namespace

namespace mshbm {
// error text for calls without a context (codecs, create)
void set_global_error(const std::string& msg) { g_err = msg; }
}  // namespace mshbm

namespace {

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct LevelBuf {
  int h = 0, w = 0, d = 0, b = 0;
  int64_t ld = 0;
  double* L = nullptr;
  double* R = nullptr;
  float* muR = nullptr;
  float* isR = nullptr;
  float* muL = nullptr;     // left window statistics (sweep4 levels, b >= 5)
  float* isL = nullptr;
  unsigned* flags = nullptr;  // sweep4 precision-guard tile flags
  float* guard_col = nullptr; // guard scratch (per tile row and column)
  int64_t flags_ld = 0;
  int* fix_list = nullptr;   // sweep2 fixup jobs (+ count)
  int* fix_count = nullptr;
  int* wc = nullptr;
  int16_t* dsel = nullptr;
  int16_t* dmed = nullptr;
  float* c = nullptr;
  uint8_t* low = nullptr;
  double* coef = nullptr;   // spline coefficients of this level's cost map
  int64_t ldc = 0;
  float* Rp = nullptr;      // padded staging arrays of the sweep (prep_staging)
  float2* Mp = nullptr;
  int64_t ldp = 0;
  int pc = 0;
  RowBand rows{0, 0, 0, 0};  // sweep/prior/median rows and counted rows
  // rows of the level image (img) and of its statistics / staging arrays (st)
  // the rows above need: whole level, or a row band's share plus halos
  int img_lo = 0, img_hi = 0, st_lo = 0, st_hi = 0;
};

struct PlanKey {
  int H, W, K, user, band_lo, band_hi, slot;
  int d_max, block, radius, sign;
  double alpha, beta, eps;
  std::vector<int> lvl;     // per-level (h, w, d, b) for user pyramids
  bool operator<(const PlanKey& o) const {
    return std::tie(H, W, K, user, band_lo, band_hi, slot, d_max, block, radius, sign, alpha,
                    beta, eps, lvl) <
           std::tie(o.H, o.W, o.K, o.user, o.band_lo, o.band_hi, o.slot, o.d_max, o.block,
                    o.radius, o.sign, o.alpha, o.beta, o.eps, o.lvl);
  }
};

struct StageEvents {
  cudaEvent_t up0, up1, sel0, sel1, med0, med1;
};

struct Plan {
  PlanKey key{};
  int H = 0, W = 0, K = 0;
  bool user = false;
  // level 0 kept as an fp64 copy (caller-supplied pyramid, no pyramid, or a
  // block only the generic fp64 sweep handles); otherwise every level-0
  // kernel reads the fp32 inputs and the copy is never written
  bool l0_f64 = true;
  mshbm_config cfg{};
  std::vector<LevelBuf> lv;
  float* in_l = nullptr;
  float* in_r = nullptr;
  int64_t ld_in = 0;
  unsigned long long* counters = nullptr;
  float* cR = nullptr;        // right-image offset c of every level (centre sample)
  void* arena = nullptr;
  cudaGraphExec_t exec = nullptr;         // plain graph
  cudaGraphExec_t exec_timed = nullptr;   // + the stage event-record nodes
  int launches = 0;
  // host-output streaming (run_plan_io, launch_streamed): everything up to
  // level 0's prior as one graph, then level 0's selection + median in row
  // chunks, each chunk's rows copied to the host while the next one runs
  cudaGraphExec_t exec_pre = nullptr;
  std::vector<cudaGraphExec_t> exec_l0;
  std::vector<int> l0_cut;                // chunk i = output rows [l0_cut[i], l0_cut[i + 1])
  std::vector<cudaEvent_t> l0_ev;         // chunk i's median done
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_done = nullptr;
  int launches_streamed = 0;
  cudaStream_t stream = nullptr;   // batch slot stream (run_batch)
  // recorded after every use: a call on another stream waits for it before
  // touching the plan's buffers (inputs, pyramid, outputs are per plan)
  cudaEvent_t done = nullptr;
  cudaStream_t last_stream = nullptr;
  bool used = false;
  // stage timing: events recorded by every run (external event-record nodes
  // of the captured graph, or plain records on the direct path)
  std::vector<StageEvents> tev;
  cudaEvent_t t_begin = nullptr, t_built = nullptr, t_end = nullptr;
};

}  // namespace

struct mshbm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::recursive_mutex mu;   // plans map + plan use (calls from several host threads)
  std::map<PlanKey, Plan*> plans;
  int64_t launches = 0;
  cudaEvent_t ev[64];
  int n_ev = 0;
};

struct mshbm_engine {
  mshbm_ctx* ctx = nullptr;
  int H = 0, W = 0, d = 0, b = 0, dir = 1;
  double eps = 1e-6;
  int64_t ld = 0;
  double *L = nullptr, *R = nullptr;
  double *muL = nullptr, *sgL = nullptr, *muR = nullptr, *sgR = nullptr;
  float *muR32 = nullptr, *isR32 = nullptr;
  float* Rp = nullptr;
  float2* Mp = nullptr;
  int64_t ldp = 0;
  int pc = 0;
  int* wc = nullptr;
  int16_t *fz = nullptr, *wz = nullptr, *nz = nullptr;
  float *fc = nullptr, *wcst = nullptr, *nc = nullptr;
  unsigned long long* counters = nullptr;
  int* bad = nullptr;
  void* arena = nullptr;
};

namespace {

int fail(mshbm_ctx* ctx, int code, const std::string& msg) {
  g_err = msg;
  if (ctx) ctx->err = msg;
  return code;
}

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(ctx, MSHBM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// NULL selects the legacy default stream (CUDA's own convention), so calls
// from torch's default stream stay ordered with torch's work.
cudaStream_t pick(mshbm_ctx*, void* s) { return (cudaStream_t)s; }

// ---------------------------------------------------------------- config
int validate_config(mshbm_ctx* ctx, const mshbm_config* c) {
  char buf[160];
  if (!c) return fail(ctx, MSHBM_ERR_CONFIG, "null config");
  if (c->d_max < 1) {
    snprintf(buf, sizeof buf, "d_max must be >= 1, got %d", c->d_max);
    return fail(ctx, MSHBM_ERR_CONFIG, buf);
  }
  if (c->block < 3 || c->block % 2 == 0) {
    snprintf(buf, sizeof buf, "block must be odd and >= 3, got %d", c->block);
    return fail(ctx, MSHBM_ERR_CONFIG, buf);
  }
  if (!(c->alpha > 0.0 && c->alpha < 1.0)) {
    snprintf(buf, sizeof buf, "alpha must lie in (0, 1), got %g", c->alpha);
    return fail(ctx, MSHBM_ERR_CONFIG, buf);
  }
  if (!(c->beta > 0.0 && c->beta < 1.0)) {
    snprintf(buf, sizeof buf, "beta must lie in (0, 1), got %g", c->beta);
    return fail(ctx, MSHBM_ERR_CONFIG, buf);
  }
  if (!(c->sigma_eps > 0.0)) {
    snprintf(buf, sizeof buf, "sigma_eps must be positive, got %g", c->sigma_eps);
    return fail(ctx, MSHBM_ERR_CONFIG, buf);
  }
  if (c->sign != MSHBM_SIGN_MIDDLEBURY && c->sign != MSHBM_SIGN_PAPER)
    return fail(ctx, MSHBM_ERR_CONFIG, "unknown sign convention");
  if (c->radius < 0) return fail(ctx, MSHBM_ERR_CONFIG, "radius must be >= 0");
  return MSHBM_OK;
}

// ---------------------------------------------------------------- plans
struct Carver {
  size_t off = 0;
  char* base = nullptr;
  template <typename T>
  T* take(size_t n) {
    off = (size_t)round_up((int64_t)off, 256);
    T* p = base ? (T*)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

// Whether the level-0-style sweep4 will run on this level (then it needs the
// left statistics, the guard flags and the fixup job list).
bool level_uses_sweep4(const Plan& p, const LevelBuf& l) {
  SweepArgs a{};
  a.H = l.h; a.W = l.w; a.d = l.d; a.block = l.b; a.dir = p.cfg.sign == MSHBM_SIGN_PAPER ? -1 : 1;
  a.mode = kSweepPipeline;
  static float f1;
  static unsigned f2;
  a.muL = &f1; a.isL = &f1; a.tile_flags = &f2;   // non-null stand-ins for the query
  return sweep_uses_sweep4(a);
}

void carve(Plan& p, Carver& cv) {
  const int64_t ldi = round_up(p.W, 32);
  p.ld_in = ldi;
  p.in_l = cv.take<float>((size_t)ldi * p.H);
  p.in_r = cv.take<float>((size_t)ldi * p.H);
  p.counters = cv.take<unsigned long long>((size_t)(p.K + 1) * kCntSlots * kCntCopies);
  p.cR = cv.take<float>(1);
  for (auto& l : p.lv) {
    const size_t n = (size_t)l.ld * l.h;
    l.L = cv.take<double>(n);
    l.R = cv.take<double>(n);
    l.muR = cv.take<float>(n);
    l.isR = cv.take<float>(n);
    if (level_uses_sweep4(p, l)) {
      l.muL = cv.take<float>(n);
      l.isL = cv.take<float>(n);
      // one word per 16-column x (>= 2)-row tile (sweep4_th() >= 2), then the
      // fixup job count (zeroed together before every run)
      l.flags_ld = (l.w + 15) / 16;
      l.flags = cv.take<unsigned>((size_t)l.flags_ld * ((l.h + 1) / 2) + 1);
      l.fix_count = reinterpret_cast<int*>(l.flags + (size_t)l.flags_ld * ((l.h + 1) / 2));
      l.fix_list = cv.take<int>((size_t)((l.w + 29) / 30) * (l.h / 14 + 2));
      l.guard_col = cv.take<float>((size_t)((l.h + sweep4_th() - 1) / sweep4_th() + 1) * l.w);
    }
    l.wc = cv.take<int>(n);
    l.dsel = cv.take<int16_t>(n);
    l.dmed = cv.take<int16_t>(n);
    l.c = cv.take<float>(n);
    l.low = cv.take<uint8_t>(n);
    l.ldc = round_up(l.w + 24, 32);
    l.coef = cv.take<double>((size_t)l.ldc * (l.h + 24));
    l.pc = staging_margin(l.d, l.b);
    l.ldp = round_up(l.w + 2 * l.pc, 32);
    l.Rp = cv.take<float>((size_t)l.ldp * l.h);
    l.Mp = cv.take<float2>((size_t)l.ldp * l.h);
  }
}

int build_plan(mshbm_ctx* ctx, Plan& p) {
  for (const LevelBuf& l : p.lv) {
    // the sweep addresses its staging arrays with 32-bit element offsets
    const int64_t ldp = round_up(l.w + 2 * staging_margin(l.d, l.b), 32);
    if (ldp * l.h >= ((int64_t)1 << 31))
      return fail(ctx, MSHBM_ERR_UNSUPPORTED, "level too large for 32-bit staging offsets");
  }
  Carver probe;
  carve(p, probe);
  CK(cudaMalloc(&p.arena, probe.off + 256));
  // finite contents everywhere: band runs prefilter rows they never sweep
  CK(cudaMemset(p.arena, 0, probe.off + 256));
  Carver real;
  real.base = (char*)p.arena;
  carve(p, real);
  return MSHBM_OK;
}

// Row ranges per level for a level-0 band [b0, b1) (whole image: b0=0,
// b1=H).  Level k sweeps rows S_k; level k+1 must provide exact disparities
// for rows S_k/2 and exact costs within the kCoarseHalo-row reach of the tiled
// spline prefilter + support around them.
// Coarse-level halo (rows of level k+1 beyond half of level k's rows): the
// finer level's prior reads the spline coefficients of rows [lo/2 - 2,
// hi/2 + 3] (+12 padded), each a 57-tap FIR (+-28 rows) of the coarse costs,
// and the 2x NN disparity of rows [lo/2, hi/2] from the coarse median (+-2
// rows of sweep output): <= 33 rows, 40 with margin.
constexpr int kCoarseHalo = 40;

void plan_rows(Plan& p, int b0, int b1) {
  const int K = p.K;
  for (int k = 0; k <= K; ++k) {
    LevelBuf& l = p.lv[k];
    const int own_lo = b0 >> k;
    const int own_hi = (b1 >= p.H) ? l.h : std::min(l.h, b1 >> k);
    if (k == 0) {
      l.rows.lo = std::max(0, b0 - 2);
      l.rows.hi = std::min(l.h, b1 + 2);
    } else {
      const RowBand& f = p.lv[k - 1].rows;
      l.rows.lo = std::max(0, (f.lo >> 1) - kCoarseHalo);
      l.rows.hi = std::min(l.h, (f.hi >> 1) + kCoarseHalo + 1);
    }
    l.rows.cnt_lo = own_lo;
    l.rows.cnt_hi = own_hi;
  }
  // Statistics and staging rows: the sweep's CTA grids (sweep2 jobs of <= 30
  // rows, sweep4 tiles of 32) and window halos reach <= 37 rows beyond its
  // rows; the image rows add the statistics kernel's 32-row tile alignment
  // (its tiles read, and centre on, their first row) and window (<= 5 + 31 +
  // 5 rows beyond the statistics rows), and every level must also hold the
  // rows the next coarser level's 5-tap downsample reads (2 x its rows +- 2).
  // Whole-image plans get whole levels.
  for (int k = K; k >= 0; --k) {
    LevelBuf& l = p.lv[k];
    l.st_lo = std::max(0, l.rows.lo - 40);
    l.st_hi = std::min(l.h, l.rows.hi + 40);
    l.img_lo = std::max(0, l.rows.lo - 88);
    l.img_hi = std::min(l.h, l.rows.hi + 88);
    if (k < K) {
      const LevelBuf& c = p.lv[k + 1];
      l.img_lo = std::max(0, std::min(l.img_lo, 2 * c.img_lo - 3));
      l.img_hi = std::min(l.h, std::max(l.img_hi, 2 * c.img_hi + 3));
    }
  }
}

// Event record that becomes an event-record node under stream capture.
// Untimed graphs leave them out (each node adds scheduling latency on the
// critical path of a short pipeline, ~0.1 ms on C2): g_rec_events is false
// while those are captured.
thread_local bool g_rec_events = true;
cudaError_t rec(cudaEvent_t e, cudaStream_t s) {
  if (!g_rec_events) return cudaSuccess;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t err = cudaStreamIsCapturing(s, &cs);
  if (err != cudaSuccess) return err;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}

// Enqueue the whole pair on `s` (also used under stream capture).
// side/evs (graph capture only): the window statistics and staging arrays
// of levels K-1..0 run on a forked branch, so they overlap the coarse
// levels' matching (which leaves most SMs idle); level k's sweep joins on
// evs[k].  evs[K+1] is the fork point.  The spline prefilter of level k's
// costs also runs on the branch, beside level k's median (evs[K+2+k] =
// sweep k done, evs[2K+3+(k-1)] = prefilter done, joined by prior k-1).
// Every run records the plan's stage events (p.tev, t_begin/t_built/t_end).
// part: kAll, or kPre = everything before level 0's selection (its prior
// included), or kL0 = level 0's selection + median only, on the rows of
// `chunk` (sweep rows, rows.lo..hi; median rows, cnt_lo..cnt_hi; first: the
// chunk that also runs the whole image's guard fixup).
enum { kAll = 0, kPre = 1, kL0 = 2 };
struct L0Chunk {
  RowBand sweep, median;
  bool first;
};
int enqueue(mshbm_ctx* ctx, Plan& p, cudaStream_t s, cudaStream_t side = nullptr,
            cudaEvent_t* evs = nullptr, cudaStream_t side2 = nullptr, int part = kAll,
            const L0Chunk* chunk = nullptr) {
  int n = 0;
  const mshbm_config& cfg = p.cfg;
  const int dir = cfg.sign == MSHBM_SIGN_PAPER ? -1 : 1;
  if (part != kL0) {
  CK(rec(p.t_begin, s));
  CK(cudaMemsetAsync(p.counters, 0,
                     sizeof(unsigned long long) * (p.K + 1) * kCntSlots * kCntCopies, s));
  if (!p.user) {
    if (p.K == 0) {
      CK(launch_f32_to_f64(p.in_l, p.in_r, p.H, p.W, p.ld_in, p.lv[0].L, p.lv[0].R, p.lv[0].ld,
                           s));
    } else {
      // level 1 straight from the fp32 input; also writes the fp64 level 0
      // (rows 2 i, 2 i + 1 of every level-1 row i computed)
      const LevelBuf& l0 = p.lv[0];
      const LevelBuf& l1 = p.lv[1];
      CK(launch_downsample_f32(p.in_l, p.in_r, p.H, p.W, p.ld_in, l1.L, l1.R, l1.ld,
                               p.l0_f64 ? l0.L : nullptr, p.l0_f64 ? l0.R : nullptr, l0.ld, s,
                               std::min(l1.img_lo, l0.img_lo / 2),
                               std::max(l1.img_hi, (l0.img_hi + 1) / 2)));
    }
    ++n;
    for (int k = 2; k <= p.K; ++k) {
      const LevelBuf& a = p.lv[k - 1];
      LevelBuf& b = p.lv[k];
      CK(launch_downsample(a.L, a.R, a.h, a.w, a.ld, b.L, b.R, b.ld, s, b.img_lo, b.img_hi));
      ++n;
    }
  }
  CK(rec(p.t_built, s));   // pyramid built (build_pyramid, matcher.py:410-416)
  // the right offset c of every level: the level-0 right sample at the
  // image centre (whole input on every rank, so row bands agree)
  CK(launch_centre_sample(p.user ? nullptr : p.in_r, p.user ? p.lv[0].R : nullptr,
                          p.user ? p.lv[0].ld : p.ld_in, p.H, p.W, p.cR, s));
  ++n;
  const bool fork = side != nullptr && evs != nullptr && p.K > 0;
  if (fork) {
    CK(cudaEventRecord(evs[p.K + 1], s));
    CK(cudaStreamWaitEvent(side, evs[p.K + 1], 0));
  }
  for (int k = p.K; k >= 0; --k) {
    LevelBuf& l = p.lv[k];
    cudaStream_t t = (fork && k < p.K) ? side : s;
    // level 0 of a built pyramid reads the fp32 input (its fp64 copy is exact)
    const bool in32 = k == 0 && !p.l0_f64;
    if (in32) {
      CK(launch_stats_f32(p.in_r, l.h, l.w, p.ld_in, l.b, cfg.sigma_eps, l.muR, l.isR, l.ld, t,
                          l.st_lo, l.st_hi));
      CK(launch_prep_staging(p.in_r, p.ld_in, l.muR, l.isR, l.ld, l.h, l.w, l.pc, l.Rp, l.Mp,
                             l.ldp, t, l.st_lo, l.st_hi, p.cR));
    } else {
      CK(launch_stats_f32(l.R, l.h, l.w, l.ld, l.b, cfg.sigma_eps, l.muR, l.isR, l.ld, t,
                          l.st_lo, l.st_hi));
      CK(launch_prep_staging(l.R, l.ld, l.muR, l.isR, l.ld, l.h, l.w, l.pc, l.Rp, l.Mp, l.ldp, t,
                             l.st_lo, l.st_hi, p.cR));
    }
    n += 2;
    if (l.muL) {
      // L statistics + sweep4's precision guard (tile flags), then the job
      // list of its sweep2 fixup
      Sweep4Guard g;
      g.L = l.L;
      g.ld = l.ld;
      if (k == 0 && !p.l0_f64) g.L32 = p.in_l, g.ld32 = p.ld_in;
      g.muL = l.muL;
      g.isL = l.isL;
      g.muR = l.muR;
      g.isR = l.isR;
      g.lds = l.ld;
      g.cR = p.cR;
      g.h = l.h;
      g.w = l.w;
      g.d = l.d;
      g.dir = dir;
      g.tile_h = sweep4_th();
      g.colR = l.guard_col;
      g.flags = l.flags;
      g.flags_ld = l.flags_ld;
      CK(cudaMemsetAsync(l.flags, 0, sizeof(unsigned) * (l.flags_ld * ((l.h + 1) / 2) + 1), t));
      if (in32)
        CK(launch_stats_f32(p.in_l, l.h, l.w, p.ld_in, l.b, cfg.sigma_eps, l.muL, l.isL, l.ld, t,
                            l.st_lo, l.st_hi));
      else
        CK(launch_stats_f32(l.L, l.h, l.w, l.ld, l.b, cfg.sigma_eps, l.muL, l.isL, l.ld, t,
                            l.st_lo, l.st_hi));
      CK(launch_sweep4_guard(g, l.rows, t));
      CK(launch_fixup_list(l.flags, l.flags_ld, sweep4_th(), l.h, l.w, l.rows, l.b, l.fix_list,
                           l.fix_count, t));
      n += 4;
    }
    if (fork && k < p.K) CK(cudaEventRecord(evs[k], side));
  }
  }   // part != kL0
  const bool fork = part != kL0 && side != nullptr && evs != nullptr && p.K > 0;
  for (int k = part == kL0 ? 0 : p.K; k >= 0; --k) {
    LevelBuf& l = p.lv[k];
    unsigned long long* cnt = p.counters + (size_t)(p.K - k) * kCntSlots * kCntCopies;
    StageEvents* ev = &p.tev[p.K - k];
    CK(rec(ev->up0, s));
    if (k < p.K && part != kL0) {
      LevelBuf& c = p.lv[k + 1];
      if (fork) {
        CK(cudaStreamWaitEvent(s, evs[2 * p.K + 3 + k], 0));   // prefilter of level k+1
      } else {
        int r0, r1;
        prior_coef_rows(c.h, l.h, l.rows, &r0, &r1);
        CK(launch_bspline_prefilter(c.c, nullptr, c.h, c.w, c.ld, c.coef, c.ldc, s, r0, r1));
        n += 1;
      }
      CK(launch_prior_eval(c.dmed, c.ld, c.h, c.w, c.coef, c.ldc, l.h, l.w, l.d, cfg.radius,
                           cfg.beta, l.wc, l.ld, cnt, l.rows, s));
      ++n;
    }
    CK(rec(ev->up1, s));
    SweepArgs a{};
    a.L = l.L; a.R = l.R; a.ld = l.ld;
    if (k == 0 && !p.l0_f64) a.L32 = p.in_l, a.R32 = p.in_r, a.ld32 = p.ld_in;
    a.muR = l.muR; a.isR = l.isR; a.lds = l.ld;
    a.muL = l.muL; a.isL = l.isL;
    a.tile_flags = l.flags; a.flags_ld = l.flags_ld;
    a.fix_list = l.fix_list; a.fix_count = l.fix_count;
    a.H = l.h; a.W = l.w; a.d = l.d; a.block = l.b; a.dir = dir;
    a.sigma_eps = cfg.sigma_eps;
    a.wc = k < p.K ? l.wc : nullptr; a.ldw = l.ld; a.radius = cfg.radius;
    a.alpha = cfg.alpha; a.mode = kSweepPipeline;
    a.dout = l.dsel; a.cout = l.c; a.low = l.low; a.ldo = l.ld;
    a.counters = cnt;
    a.rows = l.rows;
    a.Rp = l.Rp; a.Mp = l.Mp; a.ldp = l.ldp; a.pc = l.pc;
    if (fork && k < p.K) CK(cudaStreamWaitEvent(s, evs[k], 0));
    if (part == kPre && k == 0) break;   // level 0's selection + median: the kL0 chunks
    const bool s4 = sweep_uses_sweep4(a);
    CK(rec(ev->sel0, s));
    if (part == kL0) a.rows = chunk->sweep;
    CK(launch_sweep(a, s, &n));
    if (s4 && (part != kL0 || chunk->first)) {
      // sweep2 on the tiles sweep4's precision guard left (usually none);
      // chunked runs: once, for the whole level (the job list is the whole
      // level's; it reads what sweep4 reads and writes only flagged tiles)
      a.rows = l.rows;
      CK(launch_sweep4_fixup(a, s));
      ++n;
    }
    CK(rec(ev->sel1, s));
    if (fork && k > 0) {
      // the prefilter of this level's costs (next level's prior) overlaps
      // this level's selective median
      CK(cudaEventRecord(evs[p.K + 2 + k], s));
      // (its own branch: the next level's prior waits for it, and it must not
      // queue behind the statistics branch's level-0 work)
      cudaStream_t pf = side2 ? side2 : side;
      CK(cudaStreamWaitEvent(pf, evs[p.K + 2 + k], 0));
      int r0, r1;   // the coefficient rows the next finer level's prior reads
      prior_coef_rows(l.h, p.lv[k - 1].h, p.lv[k - 1].rows, &r0, &r1);
      CK(launch_bspline_prefilter(l.c, nullptr, l.h, l.w, l.ld, l.coef, l.ldc, pf, r0, r1));
      CK(cudaEventRecord(evs[2 * p.K + 3 + (k - 1)], pf));
      n += 1;
    }
    CK(rec(ev->med0, s));
    CK(launch_median_pipeline(l.dsel, l.c, l.low, l.ld, l.h, l.w, cfg.alpha, l.dmed, cnt,
                              part == kL0 ? chunk->median : l.rows, s));
    ++n;
    CK(rec(ev->med1, s));
  }
  CK(rec(p.t_end, s));
  if (part == kAll) p.launches = n;
  else p.launches_streamed += n;
  return MSHBM_OK;
}

Plan* get_plan(mshbm_ctx* ctx, const PlanKey& key, const mshbm_config& cfg,
               const std::vector<std::tuple<int, int, int, int>>& dims, int* st) {
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) return it->second;
  Plan* p = new Plan();
  p->key = key;
  p->H = key.H;
  p->W = key.W;
  p->K = key.K;
  p->user = key.user != 0;
  p->cfg = cfg;
  for (auto& t : dims) {
    LevelBuf l;
    l.h = std::get<0>(t);
    l.w = std::get<1>(t);
    l.d = std::get<2>(t);
    l.b = std::get<3>(t);
    l.ld = round_up(l.w, 32);
    p->lv.push_back(l);
  }
  p->l0_f64 = p->user || p->K == 0 || p->lv[0].b > 11;
  *st = build_plan(ctx, *p);
  if (*st != MSHBM_OK) {
    delete p;
    return nullptr;
  }
  plan_rows(*p, key.band_lo, key.band_hi);
  p->tev.resize(p->K + 1);
  bool ok = cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t* e : {&p->t_begin, &p->t_built, &p->t_end}) ok &= cudaEventCreate(e) == cudaSuccess;
  for (auto& e : p->tev) {
    cudaEvent_t* ev = &e.up0;
    for (int t = 0; t < 6; ++t) ok &= cudaEventCreate(&ev[t]) == cudaSuccess;
  }
  if (!ok) {
    *st = fail(ctx, MSHBM_ERR_CUDA, "event create failed");
    return nullptr;
  }
  ctx->plans[key] = p;
  return p;
}

// run a plan: graph replay (captured on first use) or direct launches
// (MSHBM_FLAG_NO_GRAPH).  Direct launches and timed replays
// (MSHBM_FLAG_TIMING) record the plan's stage events; untimed replays use a
// graph without them.
int launch_plan(mshbm_ctx* ctx, Plan& p, cudaStream_t s, int flags) {
  if (flags & MSHBM_FLAG_NO_GRAPH) {
    int st = enqueue(ctx, p, s);
    if (st) return st;
  } else {
    const bool timed = (flags & MSHBM_FLAG_TIMING) != 0;
    cudaGraphExec_t& exec = timed ? p.exec_timed : p.exec;
    if (!exec) {
      cudaStream_t cs;
      CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      cudaStream_t side, side2;
      CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
      std::vector<cudaEvent_t> evs(3 * p.K + 4);
      for (auto& e : evs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      // prefilters get their own branch only when the statistics branch
      // carries sweep4's extra level-0 work (measured: small pipelines are
      // faster with one branch)
      bool s4 = false;
      for (const LevelBuf& l : p.lv) s4 |= l.muL != nullptr;
      g_rec_events = timed;
      int st = enqueue(ctx, p, cs, side, evs.data(), s4 ? side2 : nullptr);
      g_rec_events = true;
      cudaError_t ce = cudaStreamEndCapture(cs, &g);
      for (auto& e : evs) cudaEventDestroy(e);
      cudaStreamDestroy(side);
      cudaStreamDestroy(side2);
      cudaStreamDestroy(cs);
      if (st) return st;
      CK(ce);
      CK(cudaGraphInstantiate(&exec, g, 0));
      cudaGraphDestroy(g);
    }
    CK(cudaGraphLaunch(exec, s));
  }
  ctx->launches += p.launches;
  return MSHBM_OK;
}

// Host-output streaming (MSHBM_IO_HOST, untimed, whole image): level 0's
// selection + median run in row chunks after the rest of the pair, and each
// chunk's disparity / cost rows go to the host on a copy stream while the
// next chunk computes, so only the last chunk's copy is exposed.  Chunk
// boundaries sit 4 rows above a sweep4 tile row (sweep rows [cut + 2, next
// cut + 2) are whole tiles of the offset tile grid: no tile is swept twice),
// chunks write disjoint rows, and every kernel keeps its whole-image tile
// grid, so the outputs are bit-identical to the one-graph path (row bands'
// property).
bool stream_eligible(const Plan& p) {
  static const int on = []() {
    const char* v = getenv("MSHBM_STREAM_L0");
    return v ? atoi(v) : 1;
  }();
  if (!on || p.user || p.K < 1) return false;
  if (p.key.band_lo != 0 || p.key.band_hi < p.H) return false;
  const LevelBuf& l0 = p.lv[0];
  // a sweep4 level 0 tall enough that a chunk's tiles still fill the GPU
  return l0.muL != nullptr && l0.h >= 1024;
}

int capture_part(mshbm_ctx* ctx, Plan& p, int part, const L0Chunk* chunk, cudaGraphExec_t* exec) {
  cudaStream_t cs, side, side2;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> evs(3 * p.K + 4);
  for (auto& e : evs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  g_rec_events = false;
  int st = part == kL0 ? enqueue(ctx, p, cs, nullptr, nullptr, nullptr, kL0, chunk)
                       : enqueue(ctx, p, cs, side, evs.data(), side2, part, nullptr);
  g_rec_events = true;
  cudaError_t ce = cudaStreamEndCapture(cs, &g);
  for (auto& e : evs) cudaEventDestroy(e);
  cudaStreamDestroy(side);
  cudaStreamDestroy(side2);
  cudaStreamDestroy(cs);
  if (st) return st;
  CK(ce);
  CK(cudaGraphInstantiate(exec, g, 0));
  cudaGraphDestroy(g);
  return MSHBM_OK;
}

int launch_streamed(mshbm_ctx* ctx, Plan& p, cudaStream_t s, int16_t* disparity, float* cost,
                    int64_t ld_out) {
  const LevelBuf& l0 = p.lv[0];
  if (!p.exec_pre) {
    // chunk cuts: multiples of the tile height minus 4 (see above)
    const int th = sweep4_th();
    static const int want = []() {
      const char* v = getenv("MSHBM_STREAM_CHUNKS");
      return v ? std::max(1, atoi(v)) : 4;
    }();
    std::vector<int> cut{0};
    // shrinking chunks: a copy takes about a third of the time its rows took to
    // compute, so every chunk still hides the previous one's copy, and the
    // last chunk's copy, the exposed one, is small
    std::vector<double> frac;
    if (const char* v = getenv("MSHBM_STREAM_CUTS")) {
      for (const char* q = v; *q;) {
        frac.push_back(atof(q));
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    } else if (want == 4) {
      frac = {0.4, 0.7, 0.9};   // measured best on C3 (4.20 ms; uniform quarters 4.29)
    } else {
      double left = 1.0, at = 0.0;
      for (int i = 1; i < want; ++i) {
        at += left * 0.45;
        left *= 0.55;
        frac.push_back(at);
      }
    }
    for (double f : frac) {
      const int c = (int)((l0.h * f + th / 2) / th) * th - 4;
      if (c > cut.back() + th && c < l0.h - th) cut.push_back(c);
    }
    cut.push_back(l0.h);
    p.launches_streamed = 0;
    int st = capture_part(ctx, p, kPre, nullptr, &p.exec_pre);
    if (st) return st;
    const int nc = (int)cut.size() - 1;
    p.exec_l0.assign(nc, nullptr);
    for (int i = 0; i < nc; ++i) {
      L0Chunk ch;
      const int lo = i == 0 ? 0 : cut[i] + 2, hi = i == nc - 1 ? l0.h : cut[i + 1] + 2;
      ch.sweep = RowBand{lo, hi, lo, hi};
      ch.median = RowBand{cut[i], cut[i + 1], cut[i], cut[i + 1]};
      ch.first = i == 0;
      st = capture_part(ctx, p, kL0, &ch, &p.exec_l0[i]);
      if (st) return st;
    }
    p.l0_ev.resize(nc);
    for (auto& e : p.l0_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p.copy_done, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&p.copy_stream, cudaStreamNonBlocking));
    p.l0_cut = cut;
  }
  CK(cudaGraphLaunch(p.exec_pre, s));
  const int nc = (int)p.exec_l0.size();
  // every chunk is enqueued before the first copy: a copy into pageable host
  // memory blocks the calling thread, and must not hold back the launches
  for (int i = 0; i < nc; ++i) {
    CK(cudaGraphLaunch(p.exec_l0[i], s));
    CK(cudaEventRecord(p.l0_ev[i], s));
  }
  for (int i = 0; i < nc; ++i) {
    CK(cudaStreamWaitEvent(p.copy_stream, p.l0_ev[i], 0));
    const int r0 = p.l0_cut[i], nr = p.l0_cut[i + 1] - r0;
    if (disparity)
      CK(cudaMemcpy2DAsync(disparity + (int64_t)r0 * ld_out, ld_out * 2,
                           l0.dmed + (int64_t)r0 * l0.ld, l0.ld * 2, (size_t)l0.w * 2, nr,
                           cudaMemcpyDeviceToHost, p.copy_stream));
    if (cost)
      CK(cudaMemcpy2DAsync(cost + (int64_t)r0 * ld_out, ld_out * 4, l0.c + (int64_t)r0 * l0.ld,
                           l0.ld * 4, (size_t)l0.w * 4, nr, cudaMemcpyDeviceToHost,
                           p.copy_stream));
  }
  CK(cudaEventRecord(p.copy_done, p.copy_stream));
  CK(cudaStreamWaitEvent(s, p.copy_done, 0));
  ctx->launches += p.launches_streamed;
  return MSHBM_OK;
}

// Pack host copies of the device counters into LevelTrace records exactly as
// run_pipeline fills them (matcher.py:377-463).
// sum (window max: max) the kCntCopies copies of one level's counters
void reduce_copies(const unsigned long long* h, unsigned long long* c) {
  for (int s = 0; s < kCntSlots; ++s) c[s] = 0;
  for (int cp = 0; cp < kCntCopies; ++cp)
    for (int s = 0; s < kCntSlots; ++s) {
      const unsigned long long v = h[(size_t)cp * kCntSlots + s];
      c[s] = s == kCntWindowMax ? std::max(c[s], v) : c[s] + v;
    }
}

void pack_trace(const Plan& p, const unsigned long long* h, mshbm_level_trace* trace,
                bool timed) {
  float ms_build = 0.f, ms_total = 0.f;
  if (timed) {
    cudaEventElapsedTime(&ms_build, p.t_begin, p.t_built);
    cudaEventElapsedTime(&ms_total, p.t_begin, p.t_end);
  }
  for (int t = 0; t <= p.K; ++t) {
    const int k = p.K - t;
    const LevelBuf& l = p.lv[k];
    unsigned long long c[kCntSlots];
    reduce_copies(&h[(size_t)t * kCntSlots * kCntCopies], c);
    mshbm_level_trace& o = trace[t];
    memset(&o, 0, sizeof o);
    o.level = k;
    o.height = l.h;
    o.width = l.w;
    o.d_max = l.d;
    o.block = l.b;
    const int64_t N = (int64_t)(l.rows.cnt_hi - l.rows.cnt_lo) * l.w;
    if (k == p.K) {
      o.full_search_pixels = N;
      o.selection_evals = N * (l.d + 1);
    } else {
      o.trusted = (int64_t)c[kCntTrusted];
      o.trusted_evals = (int64_t)c[kCntTrustedEvals];
      o.trusted_window_max = (int64_t)c[kCntWindowMax];
      o.full_search_pixels = N - o.trusted;
      o.selection_evals = o.trusted_evals + o.full_search_pixels * (l.d + 1);
    }
    o.refined = (int64_t)c[kCntRefined];
    o.refine_evals = o.refined > 0 ? (int64_t)c[kCntNeeded] * (l.d + 1) : 0;
    o.median_replaced = (int64_t)c[kCntMedianReplaced];
    if (timed) {
      const StageEvents& e = p.tev[t];
      float ms = 0.f;
      if (k < p.K) {
        cudaEventElapsedTime(&ms, e.up0, e.up1);
        o.ms_upsample = ms;
      }
      cudaEventElapsedTime(&ms, e.sel0, e.sel1);
      o.ms_select = ms;
      o.ms_refine = 0.f;   // fused into the sweep (reported under select)
      cudaEventElapsedTime(&ms, e.med0, e.med1);
      o.ms_median = ms;
      o.ms_build = ms_build;
      o.ms_total = ms_total;
    }
  }
}

// Copy the device counters back (synchronises `s`) and pack the trace.
int finish_trace(mshbm_ctx* ctx, Plan& p, cudaStream_t s, mshbm_level_trace* trace, bool timed) {
  std::vector<unsigned long long> h((size_t)(p.K + 1) * kCntSlots * kCntCopies);
  CK(cudaMemcpyAsync(h.data(), p.counters, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  pack_trace(p, h.data(), trace, timed);
  return MSHBM_OK;
}

void destroy_events(std::vector<StageEvents>& tev) {
  for (auto& e : tev) {
    cudaEvent_t* ev = &e.up0;
    for (int t = 0; t < 6; ++t) cudaEventDestroy(ev[t]);
  }
  tev.clear();
}

// A plan's buffers belong to one stream at a time: a call on a different
// stream than the plan's last user waits for that use to finish.
int plan_acquire(mshbm_ctx* ctx, Plan& p, cudaStream_t s) {
  if (p.used && p.last_stream != s) CK(cudaStreamWaitEvent(s, p.done, 0));
  return MSHBM_OK;
}
int plan_release(mshbm_ctx* ctx, Plan& p, cudaStream_t s) {
  CK(cudaEventRecord(p.done, s));
  p.last_stream = s;
  p.used = true;
  return MSHBM_OK;
}

// inputs (optional) -> plan -> outputs (+ trace).  Host I/O synchronises.
int run_plan_io(mshbm_ctx* ctx, Plan* p, const float* left, const float* right, int64_t ld,
                int16_t* disparity, float* cost, int64_t ld_out, mshbm_level_trace* trace,
                int32_t io, int32_t flags, cudaStream_t s, bool allow_sync = true) {
  const bool host = io == MSHBM_IO_HOST;
  const cudaMemcpyKind kin = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const cudaMemcpyKind kout = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  int st = plan_acquire(ctx, *p, s);
  if (st) return st;
  if (left) {
    CK(cudaMemcpy2DAsync(p->in_l, p->ld_in * 4, left, ld * 4, (size_t)p->W * 4, p->H, kin, s));
    CK(cudaMemcpy2DAsync(p->in_r, p->ld_in * 4, right, ld * 4, (size_t)p->W * 4, p->H, kin, s));
  }
  if (host && allow_sync && flags == 0 && trace == nullptr && (disparity || cost) &&
      stream_eligible(*p)) {
    st = launch_streamed(ctx, *p, s, disparity, cost, ld_out);
    if (st) return st;
    st = plan_release(ctx, *p, s);
    if (st) return st;
    CK(cudaStreamSynchronize(s));
    return MSHBM_OK;
  }
  st = launch_plan(ctx, *p, s, flags);
  if (st) return st;
  const LevelBuf& l0 = p->lv[0];
  const int r0 = l0.rows.cnt_lo, nr = l0.rows.cnt_hi - l0.rows.cnt_lo;
  if (disparity)
    CK(cudaMemcpy2DAsync(disparity, ld_out * 2, l0.dmed + (int64_t)r0 * l0.ld, l0.ld * 2,
                         (size_t)l0.w * 2, nr, kout, s));
  if (cost)
    CK(cudaMemcpy2DAsync(cost, ld_out * 4, l0.c + (int64_t)r0 * l0.ld, l0.ld * 4,
                         (size_t)l0.w * 4, nr, kout, s));
  st = plan_release(ctx, *p, s);
  if (st) return st;
  if (trace) st = finish_trace(ctx, *p, s, trace, (flags & MSHBM_FLAG_TIMING) != 0);
  else if (host && allow_sync) {
    CK(cudaStreamSynchronize(s));
  }
  return st;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

int mshbm_abi_version(void) { return MSHBM_ABI_VERSION; }

const char* mshbm_status_string(int s) {
  switch (s) {
    case MSHBM_OK: return "ok";
    case MSHBM_ERR_VALUE: return "value error";
    case MSHBM_ERR_CONFIG: return "config error";
    case MSHBM_ERR_CUDA: return "cuda error";
    case MSHBM_ERR_NOMEM: return "out of memory";
    case MSHBM_ERR_UNSUPPORTED: return "unsupported";
    case MSHBM_ERR_DECODE: return "decode error";
    case MSHBM_ERR_MALFORMED: return "malformed header";
    case MSHBM_ERR_TRUNCATED: return "truncated payload";
    case MSHBM_ERR_MAXVAL: return "unsupported maxval";
    case MSHBM_ERR_MISSING_KEY: return "missing key";
    default: return "unknown";
  }
}

const char* mshbm_last_error(const mshbm_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

int mshbm_create(mshbm_ctx** out, int device) {
  mshbm_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, MSHBM_ERR_VALUE, "null out pointer");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(nullptr, MSHBM_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(nullptr, MSHBM_ERR_VALUE, "bad device index");
  CK(cudaSetDevice(device));
  ctx = new mshbm_ctx();
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, MSHBM_ERR_CUDA, "stream create failed");
  }
  *out = ctx;
  return MSHBM_OK;
}

int mshbm_destroy(mshbm_ctx* ctx) {
  if (!ctx) return MSHBM_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->plans) {
    if (kv.second->exec) cudaGraphExecDestroy(kv.second->exec);
    if (kv.second->exec_timed) cudaGraphExecDestroy(kv.second->exec_timed);
    if (kv.second->exec_pre) cudaGraphExecDestroy(kv.second->exec_pre);
    for (cudaGraphExec_t e : kv.second->exec_l0)
      if (e) cudaGraphExecDestroy(e);
    for (cudaEvent_t e : kv.second->l0_ev)
      if (e) cudaEventDestroy(e);
    if (kv.second->copy_done) cudaEventDestroy(kv.second->copy_done);
    if (kv.second->copy_stream) cudaStreamDestroy(kv.second->copy_stream);
    if (kv.second->stream) cudaStreamDestroy(kv.second->stream);
    if (kv.second->done) cudaEventDestroy(kv.second->done);
    destroy_events(kv.second->tev);
    for (cudaEvent_t e : {kv.second->t_begin, kv.second->t_built, kv.second->t_end})
      if (e) cudaEventDestroy(e);
    cudaFree(kv.second->arena);
    delete kv.second;
  }
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return MSHBM_OK;
}

int64_t mshbm_launch_count(const mshbm_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t mshbm_level_d_max(int32_t d_max, int32_t k) {
  const int32_t v = d_max >> k;
  return v > 1 ? v : 1;
}

int32_t mshbm_level_block(int32_t base_block, int32_t k) {
  int32_t b = base_block >> k;
  if (b % 2 == 0) b -= 1;
  return b > 3 ? b : 3;
}

int mshbm_auto_levels(int64_t width, int64_t height, int64_t d_max, int64_t base_block,
                      int32_t* out_levels) {
  mshbm_ctx* ctx = nullptr;
  if (std::min(width, height) <= 0 || d_max < 1 || base_block < 1)
    return fail(ctx, MSHBM_ERR_VALUE, "width, height, d_max and base_block must be positive");
  int k = 0;
  while ((double)std::min(width, height) / std::ldexp(1.0, k + 1) >= 4.0 * (double)base_block &&
         (d_max >> (k + 1)) >= 2)
    ++k;
  *out_levels = k;
  return MSHBM_OK;
}

int mshbm_resolve_levels(const mshbm_config* cfg, int32_t height, int32_t width,
                         int32_t* out_levels) {
  mshbm_ctx* ctx = nullptr;
  int st = validate_config(nullptr, cfg);
  if (st) return st;
  if (height < 1 || width < 1) return fail(ctx, MSHBM_ERR_VALUE, "empty image");
  int32_t K = cfg->levels;
  if (K < 0) {
    st = mshbm_auto_levels(width, height, cfg->d_max, cfg->block, &K);
    if (st) return st;
  }
  if (K > 0) {
    int h = height, w = width;
    for (int t = 0; t < K; ++t) h = (h + 1) / 2, w = (w + 1) / 2;
    char buf[200];
    if (std::min(h, w) < 2 * mshbm_level_block(cfg->block, K)) {
      snprintf(buf, sizeof buf,
               "%d levels leave a %dx%d coarsest image, smaller than twice its %d-pixel block",
               K, h, w, mshbm_level_block(cfg->block, K));
      return fail(ctx, MSHBM_ERR_VALUE, buf);
    }
    if ((cfg->d_max >> K) < 2) {
      snprintf(buf, sizeof buf, "%d levels shrink the disparity range below 2 (d_max=%d)", K,
               cfg->d_max);
      return fail(ctx, MSHBM_ERR_VALUE, buf);
    }
  }
  *out_levels = K;
  return MSHBM_OK;
}

int mshbm_downsample(mshbm_ctx* ctx, const double* in, int32_t h, int32_t w, int64_t ld_in,
                     double* out, int64_t ld_out, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  if (h < 2 || w < 2) return fail(ctx, MSHBM_ERR_VALUE, "cannot downsample image smaller than 2x2");
  CK(cudaSetDevice(ctx->device));
  CK(launch_downsample(in, nullptr, h, w, ld_in, out, nullptr, ld_out, pick(ctx, stream)));
  ctx->launches += 1;
  return MSHBM_OK;
}

int mshbm_binomial_smooth(mshbm_ctx* ctx, const double* in, int32_t h, int32_t w,
                          int64_t ld_in, double* out, int64_t ld_out, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  if (h < 1 || w < 1) return fail(ctx, MSHBM_ERR_VALUE, "cannot smooth an empty image");
  CK(cudaSetDevice(ctx->device));
  CK(launch_binomial_smooth(in, h, w, ld_in, out, ld_out, pick(ctx, stream)));
  ctx->launches += 1;
  return MSHBM_OK;
}

static int prepare_plan(mshbm_ctx* ctx, int32_t height, int32_t width, const mshbm_config* cfg,
                        int32_t band_lo, int32_t band_hi, int32_t slot, int32_t* out_levels,
                        Plan** out) {
  int K = 0;
  int st = mshbm_resolve_levels(cfg, height, width, &K);
  if (st) return fail(ctx, st, g_err);
  if (out_levels) *out_levels = K;
  if (band_lo < 0 || band_hi > height || band_lo >= band_hi)
    return fail(ctx, MSHBM_ERR_VALUE, "row band outside the image");
  const int align = 1 << K;
  if (band_lo % align != 0 || (band_hi != height && band_hi % align != 0))
    return fail(ctx, MSHBM_ERR_VALUE,
                "row band limits must be multiples of 2^levels (" + std::to_string(align) + ")");
  CK(cudaSetDevice(ctx->device));
  std::vector<std::tuple<int, int, int, int>> dims;
  int h = height, w = width;
  for (int k = 0; k <= K; ++k) {
    const int b = mshbm_level_block(cfg->block, k);
    if (!sweep_supported_block(b)) return fail(ctx, MSHBM_ERR_UNSUPPORTED, "block larger than 63");
    dims.emplace_back(h, w, mshbm_level_d_max(cfg->d_max, k), b);
    h = (h + 1) / 2;
    w = (w + 1) / 2;
  }
  PlanKey key{height, width, K, 0, band_lo, band_hi, slot, cfg->d_max, cfg->block, cfg->radius,
              cfg->sign, cfg->alpha, cfg->beta, cfg->sigma_eps, {}};
  Plan* p = get_plan(ctx, key, *cfg, dims, &st);
  if (!p) return st;
  *out = p;
  return MSHBM_OK;
}

int mshbm_run_pipeline(mshbm_ctx* ctx, const float* left, const float* right, int32_t height,
                       int32_t width, int64_t ld, const mshbm_config* cfg, int16_t* disparity,
                       float* cost, int64_t ld_out, mshbm_level_trace* trace,
                       int32_t* out_levels, int32_t io, int32_t flags, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  std::lock_guard<std::recursive_mutex> lock(ctx->mu);
  if (!left || !right) return fail(ctx, MSHBM_ERR_VALUE, "null image pointer");
  if (ld < width || ld_out < width) return fail(ctx, MSHBM_ERR_VALUE, "row stride < width");
  Plan* p = nullptr;
  int st = prepare_plan(ctx, height, width, cfg, 0, height, 0, out_levels, &p);
  if (st) return st;
  return run_plan_io(ctx, p, left, right, ld, disparity, cost, ld_out, trace, io, flags,
                     pick(ctx, stream));
}

int mshbm_run_pipeline_band(mshbm_ctx* ctx, const float* left, const float* right,
                            int32_t height, int32_t width, int64_t ld, const mshbm_config* cfg,
                            int32_t row_begin, int32_t row_end, int16_t* disparity, float* cost,
                            int64_t ld_out, mshbm_level_trace* trace, int32_t* out_levels,
                            int32_t io, int32_t flags, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  std::lock_guard<std::recursive_mutex> lock(ctx->mu);
  if (!left || !right) return fail(ctx, MSHBM_ERR_VALUE, "null image pointer");
  if (ld < width || ld_out < width) return fail(ctx, MSHBM_ERR_VALUE, "row stride < width");
  Plan* p = nullptr;
  int st = prepare_plan(ctx, height, width, cfg, row_begin, row_end, 0, out_levels, &p);
  if (st) return st;
  return run_plan_io(ctx, p, left, right, ld, disparity, cost, ld_out, trace, io, flags,
                     pick(ctx, stream));
}

int mshbm_run_batch(mshbm_ctx* ctx, int32_t n_pairs, const float* const* lefts,
                    const float* const* rights, int32_t height, int32_t width, int64_t ld,
                    const mshbm_config* cfg, int16_t* const* disparities, float* const* costs,
                    int64_t ld_out, mshbm_level_trace* traces, int32_t io, int32_t n_streams,
                    void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  std::lock_guard<std::recursive_mutex> lock(ctx->mu);
  if (n_pairs < 0 || (n_pairs > 0 && (!lefts || !rights)))
    return fail(ctx, MSHBM_ERR_VALUE, "bad pair arrays");
  if (ld < width || ld_out < width) return fail(ctx, MSHBM_ERR_VALUE, "row stride < width");
  if (n_pairs == 0) return MSHBM_OK;
  const int nslot = std::max(1, std::min(n_streams > 0 ? n_streams : 4, n_pairs));
  cudaStream_t s = pick(ctx, stream);
  std::vector<Plan*> slot(nslot, nullptr);
  int K = 0;
  for (int k = 0; k < nslot; ++k) {
    int st = prepare_plan(ctx, height, width, cfg, 0, height, 1 + k, &K, &slot[k]);
    if (st) return st;
    Plan* p = slot[k];
    if (!p->stream) CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  }
  const size_t per = (size_t)(K + 1) * kCntSlots * kCntCopies;
  unsigned long long* hc = nullptr;
  if (traces) CK(cudaMallocHost((void**)&hc, per * n_pairs * sizeof(unsigned long long)));
  cudaEvent_t start;
  CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CK(cudaEventRecord(start, s));
  for (int k = 0; k < nslot; ++k) CK(cudaStreamWaitEvent(slot[k]->stream, start, 0));
  for (int i = 0; i < n_pairs; ++i) {
    Plan* p = slot[i % nslot];
    int st = run_plan_io(ctx, p, lefts[i], rights[i], ld, disparities ? disparities[i] : nullptr,
                         costs ? costs[i] : nullptr, ld_out, nullptr, io, 0, p->stream, false);
    if (st) return st;
    if (hc)
      CK(cudaMemcpyAsync(hc + per * i, p->counters, per * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, p->stream));
  }
  for (int k = 0; k < nslot; ++k) {
    CK(cudaEventRecord(slot[k]->done, slot[k]->stream));
    CK(cudaStreamWaitEvent(s, slot[k]->done, 0));
  }
  cudaEventDestroy(start);
  if (hc || io == MSHBM_IO_HOST) CK(cudaStreamSynchronize(s));
  if (hc) {
    for (int i = 0; i < n_pairs; ++i) pack_trace(*slot[i % nslot], hc + per * i, traces + (size_t)(K + 1) * i, false);
    cudaFreeHost(hc);
  }
  return MSHBM_OK;
}

int mshbm_run_pyramid(mshbm_ctx* ctx, int32_t n_levels, const double* const* lefts,
                      const double* const* rights, const int32_t* heights,
                      const int32_t* widths, const int64_t* lds, const int32_t* d_maxs,
                      const int32_t* blocks, const mshbm_config* cfg, int16_t* disparity,
                      float* cost, int64_t ld_out, mshbm_level_trace* trace, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  std::lock_guard<std::recursive_mutex> lock(ctx->mu);
  int st = validate_config(ctx, cfg);
  if (st) return st;
  if (n_levels < 1) return fail(ctx, MSHBM_ERR_VALUE, "empty pyramid");
  CK(cudaSetDevice(ctx->device));
  std::vector<std::tuple<int, int, int, int>> dims;
  std::vector<int> flat;
  for (int k = 0; k < n_levels; ++k) {
    if (heights[k] < 1 || widths[k] < 1) return fail(ctx, MSHBM_ERR_VALUE, "empty level");
    if (blocks[k] < 3 || blocks[k] % 2 == 0 || !sweep_supported_block(blocks[k]))
      return fail(ctx, MSHBM_ERR_VALUE, "block must be odd, >= 3 and <= 63");
    if (d_maxs[k] < 0) return fail(ctx, MSHBM_ERR_VALUE, "d_max must be >= 0");
    if (k > 0 && (heights[k] != (heights[k - 1] + 1) / 2 || widths[k] != (widths[k - 1] + 1) / 2))
      return fail(ctx, MSHBM_ERR_VALUE, "pyramid levels are not dyadic");
    dims.emplace_back(heights[k], widths[k], d_maxs[k], blocks[k]);
    flat.insert(flat.end(), {heights[k], widths[k], d_maxs[k], blocks[k]});
  }
  PlanKey key{heights[0], widths[0], n_levels - 1, 1, 0, heights[0], 0, cfg->d_max, cfg->block,
              cfg->radius, cfg->sign, cfg->alpha, cfg->beta, cfg->sigma_eps, flat};
  Plan* p = get_plan(ctx, key, *cfg, dims, &st);
  if (!p) return st;
  cudaStream_t s = pick(ctx, stream);
  for (int k = 0; k < n_levels; ++k) {
    LevelBuf& l = p->lv[k];
    CK(cudaMemcpy2DAsync(l.L, l.ld * 8, lefts[k], lds[k] * 8, (size_t)l.w * 8, l.h,
                         cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpy2DAsync(l.R, l.ld * 8, rights[k], lds[k] * 8, (size_t)l.w * 8, l.h,
                         cudaMemcpyDeviceToDevice, s));
  }
  return run_plan_io(ctx, p, nullptr, nullptr, 0, disparity, cost, ld_out, trace,
                     MSHBM_IO_DEVICE, 0, s);
}

// ------------------------------------------------------------------ engine
int mshbm_engine_create(mshbm_ctx* ctx, const double* left, const double* right, int32_t height,
                        int32_t width, int64_t ld, int32_t block, int32_t d_max, double sigma_eps,
                        int32_t sign, mshbm_engine** out) {
  if (!ctx || !out) return fail(ctx, MSHBM_ERR_VALUE, "null argument");
  if (height < 1 || width < 1) return fail(ctx, MSHBM_ERR_VALUE, "empty image");
  if (block < 3 || block % 2 == 0)
    return fail(ctx, MSHBM_ERR_VALUE, "block must be odd and >= 3, got " + std::to_string(block));
  if (!sweep_supported_block(block)) return fail(ctx, MSHBM_ERR_UNSUPPORTED, "block larger than 63");
  if (d_max < 0) return fail(ctx, MSHBM_ERR_VALUE, "d_max must be >= 0, got " + std::to_string(d_max));
  if (sign != MSHBM_SIGN_MIDDLEBURY && sign != MSHBM_SIGN_PAPER)
    return fail(ctx, MSHBM_ERR_VALUE, "unknown sign convention");
  CK(cudaSetDevice(ctx->device));
  mshbm_engine* e = new mshbm_engine();
  e->ctx = ctx;
  e->H = height; e->W = width; e->d = d_max; e->b = block;
  e->dir = sign == MSHBM_SIGN_PAPER ? -1 : 1;
  e->eps = sigma_eps;
  e->ld = round_up(width, 32);
  const size_t n = (size_t)e->ld * height, nd = (size_t)height * width;
  Carver cv;
  for (int pass = 0; pass < 2; ++pass) {
    cv.off = 0;
    e->L = cv.take<double>(n); e->R = cv.take<double>(n);
    e->muL = cv.take<double>(nd); e->sgL = cv.take<double>(nd);
    e->muR = cv.take<double>(nd); e->sgR = cv.take<double>(nd);
    e->muR32 = cv.take<float>(n); e->isR32 = cv.take<float>(n);
    e->pc = staging_margin(d_max, block);
    e->ldp = round_up(width + 2 * e->pc, 32);
    e->Rp = cv.take<float>((size_t)e->ldp * height);
    e->Mp = cv.take<float2>((size_t)e->ldp * height);
    e->wc = cv.take<int>(n);
    e->fz = cv.take<int16_t>(nd); e->wz = cv.take<int16_t>(nd); e->nz = cv.take<int16_t>(nd);
    e->fc = cv.take<float>(nd); e->wcst = cv.take<float>(nd); e->nc = cv.take<float>(nd);
    e->counters = cv.take<unsigned long long>(kCntSlots * kCntCopies);
    e->bad = cv.take<int>(1);
    if (pass == 0) {
      if (cudaMalloc(&e->arena, cv.off + 256) != cudaSuccess) {
        delete e;
        return fail(ctx, MSHBM_ERR_NOMEM, "engine allocation failed");
      }
      cv.base = (char*)e->arena;
    }
  }
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpy2DAsync(e->L, e->ld * 8, left, ld * 8, (size_t)width * 8, height, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpy2DAsync(e->R, e->ld * 8, right, ld * 8, (size_t)width * 8, height, cudaMemcpyDeviceToDevice, s));
  CK(launch_stats_f64(e->L, height, width, e->ld, block, e->muL, e->sgL, s));
  CK(launch_stats_f64(e->R, height, width, e->ld, block, e->muR, e->sgR, s));
  CK(launch_stats_f32(e->R, height, width, e->ld, block, sigma_eps, e->muR32, e->isR32, e->ld, s));
  CK(launch_prep_staging(e->R, e->ld, e->muR32, e->isR32, e->ld, height, width, e->pc, e->Rp,
                         e->Mp, e->ldp, s));
  ctx->launches += 4;
  CK(cudaStreamSynchronize(s));
  *out = e;
  return MSHBM_OK;
}

int mshbm_engine_destroy(mshbm_engine* e) {
  if (!e) return MSHBM_OK;
  cudaSetDevice(e->ctx->device);
  cudaStreamSynchronize(e->ctx->stream);
  cudaFree(e->arena);
  delete e;
  return MSHBM_OK;
}

static EngineView view(const mshbm_engine* e) {
  EngineView v;
  v.L = e->L; v.R = e->R; v.ld = e->ld;
  v.muL = e->muL; v.sgL = e->sgL; v.muR = e->muR; v.sgR = e->sgR;
  v.H = e->H; v.W = e->W; v.d = e->d; v.block = e->b; v.dir = e->dir;
  v.sigma_eps = e->eps;
  return v;
}

int mshbm_engine_stats(mshbm_engine* e, double* mean_l, double* sigma_l, double* mean_r,
                       double* sigma_r, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  cudaStream_t s = pick(ctx, stream);
  const size_t bytes = (size_t)e->H * e->W * 8;
  CK(cudaStreamSynchronize(ctx->stream));
  if (mean_l) CK(cudaMemcpyAsync(mean_l, e->muL, bytes, cudaMemcpyDeviceToDevice, s));
  if (sigma_l) CK(cudaMemcpyAsync(sigma_l, e->sgL, bytes, cudaMemcpyDeviceToDevice, s));
  if (mean_r) CK(cudaMemcpyAsync(mean_r, e->muR, bytes, cudaMemcpyDeviceToDevice, s));
  if (sigma_r) CK(cudaMemcpyAsync(sigma_r, e->sgR, bytes, cudaMemcpyDeviceToDevice, s));
  return MSHBM_OK;
}

int mshbm_engine_plane(mshbm_engine* e, int32_t z, double* out, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  if (z < 0 || z > e->d)
    return fail(ctx, MSHBM_ERR_VALUE,
                "disparity " + std::to_string(z) + " outside [0, " + std::to_string(e->d) + "]");
  CK(cudaSetDevice(ctx->device));
  CK(launch_engine_plane(view(e), z, out, pick(ctx, stream)));
  ctx->launches += 1;
  return MSHBM_OK;
}

int mshbm_engine_at(mshbm_engine* e, const int64_t* rows, const int64_t* cols, const int64_t* z,
                    int64_t n, double* out, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  if (n <= 0) return MSHBM_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  CK(cudaMemsetAsync(e->bad, 0, sizeof(int), s));
  CK(launch_engine_at(view(e), rows, cols, z, n, out, e->bad, s));
  ctx->launches += 1;
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, e->bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) return fail(ctx, MSHBM_ERR_VALUE, "disparities outside [0, " + std::to_string(e->d) + "] or pixel outside the image");
  return MSHBM_OK;
}

int mshbm_engine_dsi_rows(mshbm_engine* e, const int64_t* rows, const int64_t* cols, int64_t n,
                          double* out, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  if (n <= 0) return MSHBM_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  CK(cudaMemsetAsync(e->bad, 0, sizeof(int), s));
  CK(launch_engine_dsi(view(e), rows, cols, n, out, e->bad, s));
  ctx->launches += 1;
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, e->bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) return fail(ctx, MSHBM_ERR_VALUE, "pixel outside the image");
  return MSHBM_OK;
}

static SweepArgs raw_args(mshbm_engine* e, const int* wc, int radius) {
  SweepArgs a{};
  a.L = e->L; a.R = e->R; a.ld = e->ld;
  a.muR = e->muR32; a.isR = e->isR32; a.lds = e->ld;
  a.H = e->H; a.W = e->W; a.d = e->d; a.block = e->b; a.dir = e->dir;
  a.sigma_eps = e->eps;
  a.wc = wc; a.ldw = e->W; a.radius = radius;
  a.alpha = 0.5; a.mode = kSweepRaw;
  a.fz = e->fz; a.fc = e->fc; a.wz = e->wz; a.wcst = e->wcst; a.nz = e->nz; a.nc = e->nc;
  a.rows = RowBand{0, e->H, 0, e->H};
  a.Rp = e->Rp; a.Mp = e->Mp; a.ldp = e->ldp; a.pc = e->pc;
  return a;
}

int mshbm_match_coarsest(mshbm_engine* e, double* disparity, double* cost, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  int n = 0;
  CK(launch_sweep(raw_args(e, nullptr, 0), s, &n));
  CK(launch_combine_select(nullptr, e->H, e->W, e->fz, e->fc, e->wz, e->wcst, disparity, cost, s));
  ctx->launches += n + 1;
  return MSHBM_OK;
}

int mshbm_select_with_prior(mshbm_engine* e, const double* d_hat, const double* c_hat, double beta,
                            int32_t radius, double* disparity, double* cost, int64_t* stats,
                            void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  if (radius < 0) return fail(ctx, MSHBM_ERR_VALUE, "radius must be >= 0");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  CK(cudaMemsetAsync(e->counters, 0, kCntSlots * kCntCopies * 8, s));
  CK(launch_prior_maps(d_hat, c_hat, e->H, e->W, e->d, radius, beta, e->wc, e->W, e->counters, s));
  int n = 1;
  CK(launch_sweep(raw_args(e, e->wc, radius), s, &n));
  CK(launch_combine_select(e->wc, e->H, e->W, e->fz, e->fc, e->wz, e->wcst, disparity, cost, s));
  ctx->launches += n + 1;
  std::vector<unsigned long long> hc((size_t)kCntSlots * kCntCopies);
  CK(cudaMemcpyAsync(hc.data(), e->counters, hc.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  unsigned long long h[kCntSlots];
  reduce_copies(hc.data(), h);
  const int64_t N = (int64_t)e->H * e->W;
  if (stats) {
    stats[0] = (int64_t)h[kCntTrusted];
    stats[1] = (int64_t)h[kCntTrustedEvals];
    stats[2] = (int64_t)h[kCntWindowMax];
    stats[3] = N - stats[0];
    stats[4] = stats[1] + stats[3] * (e->d + 1);
  }
  return MSHBM_OK;
}

int mshbm_refine_level(mshbm_engine* e, const double* disparity, const double* cost, double alpha,
                       double* out_disparity, double* out_cost, int64_t* evals, void* stream) {
  mshbm_ctx* ctx = e ? e->ctx : nullptr;
  if (!e) return fail(nullptr, MSHBM_ERR_VALUE, "null engine");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  CK(cudaMemsetAsync(e->counters, 0, kCntSlots * kCntCopies * 8, s));
  int n = 0;
  CK(launch_sweep(raw_args(e, nullptr, 0), s, &n));
  CK(launch_combine_refine(disparity, cost, e->H, e->W, alpha, e->nz, e->nc, out_disparity,
                           out_cost, e->counters, s));
  ctx->launches += n + 1;
  std::vector<unsigned long long> hc((size_t)kCntSlots * kCntCopies);
  CK(cudaMemcpyAsync(hc.data(), e->counters, hc.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  unsigned long long h[kCntSlots];
  reduce_copies(hc.data(), h);
  if (evals) *evals = h[kCntRefined] > 0 ? (int64_t)h[kCntNeeded] * (e->d + 1) : 0;
  return MSHBM_OK;
}

int mshbm_selective_median(mshbm_ctx* ctx, const double* disparity, const double* cost,
                           int32_t height, int32_t width, double alpha, double* out,
                           int64_t* replaced, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  if (height < 1 || width < 1) return MSHBM_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  unsigned long long* cnt = nullptr;
  CK(cudaMallocAsync((void**)&cnt, 8, s));
  CK(cudaMemsetAsync(cnt, 0, 8, s));
  CK(launch_median_f64(disparity, cost, height, width, alpha, out, cnt, s));
  ctx->launches += 1;
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(cnt, s));
  CK(cudaStreamSynchronize(s));
  if (replaced) *replaced = (int64_t)h;
  return MSHBM_OK;
}

int mshbm_upsample_prior(mshbm_ctx* ctx, const double* d_coarse, const double* c_coarse,
                         int32_t ch, int32_t cw, int32_t h, int32_t w, double* d_hat,
                         double* c_hat, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  if (ch != (h + 1) / 2 || cw != (w + 1) / 2 || ch < 1 || cw < 1) {
    char buf[160];
    snprintf(buf, sizeof buf, "%dx%d maps cannot upsample to %dx%d: not the dyadic parent", ch, cw,
             h, w);
    return fail(ctx, MSHBM_ERR_VALUE, buf);
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  const int64_t ldc = round_up(cw + 24, 32);
  double* coef = nullptr;
  CK(cudaMallocAsync((void**)&coef, (size_t)ldc * (ch + 24) * 8 * 2, s));
  CK(launch_bspline_prefilter(nullptr, c_coarse, ch, cw, cw, coef, ldc, s));
  CK(launch_upsample(d_coarse, ch, cw, coef, ldc, h, w, d_hat, c_hat, s));
  ctx->launches += 2;
  CK(cudaFreeAsync(coef, s));
  return MSHBM_OK;
}

int mshbm_evaluate(mshbm_ctx* ctx, const double* disparity, const double* gt_values,
                   const uint8_t* gt_invalid, int64_t n, double scale, const double* taus,
                   int64_t* counts, double* abs_err_sum, void* stream) {
  if (!ctx) return fail(nullptr, MSHBM_ERR_VALUE, "null context");
  if (!(scale > 0.0)) return fail(ctx, MSHBM_ERR_VALUE, "scale must be positive");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = pick(ctx, stream);
  unsigned long long* dc = nullptr;
  CK(cudaMallocAsync((void**)&dc, 7 * 8, s));
  CK(cudaMemsetAsync(dc, 0, 7 * 8, s));
  CK(launch_evaluate(disparity, gt_values, gt_invalid, n, scale, taus, dc, (double*)(dc + 6), s));
  ctx->launches += 1;
  unsigned long long h[7];
  CK(cudaMemcpyAsync(h, dc, sizeof h, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(dc, s));
  CK(cudaStreamSynchronize(s));
  for (int q = 0; q < 6; ++q) counts[q] = (int64_t)h[q];
  memcpy(abs_err_sum, &h[6], sizeof(double));
  return MSHBM_OK;
}

}  // extern "C"
