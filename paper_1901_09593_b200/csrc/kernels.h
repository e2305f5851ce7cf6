// Internal launcher interface between api.cu and the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mshbm {

// ---------------------------------------------------------------- sweep
// Dense fused ZNCC z-sweep for one level (SURVEY §7 K3a/K3b/K3c fused):
// every pixel x every z in [0, d], three register-resident winner-take-all
// states (full range, +-r prior window, 3x3-summed cost), then the
// reference's selection/refinement gates in the epilogue.
enum SweepMode { kSweepPipeline = 0, kSweepRaw = 1 };

// Row range a stage computes ([lo, hi)) and the rows whose pixels it counts
// in the trace ([cnt_lo, cnt_hi)); whole-image runs use [0, H) for both.
struct RowBand {
  int lo, hi, cnt_lo, cnt_hi;
};

struct SweepArgs {
  const double* L;      // level images, float64, row stride ld
  const double* R;
  int64_t ld;
  // level 0 of a built pyramid: the fp32 inputs (the level's values exactly;
  // its fp64 copy is then not written), row stride ld32; nullptr otherwise
  const float* L32;
  const float* R32;
  int64_t ld32;
  __host__ __device__ double Lv(int64_t y, int64_t x) const {
    return L32 ? (double)L32[y * ld32 + x] : L[y * ld + x];
  }
  __host__ __device__ double Rv(int64_t y, int64_t x) const {
    return R32 ? (double)R32[y * ld32 + x] : R[y * ld + x];
  }
  const float* muR;     // box mean of R (fp32)
  const float* isR;     // 1/sigma_R, 0 where degenerate (fp32)
  int64_t lds;
  const float* muL;     // box mean / 1/sigma of L (stride lds); sweep4 only
  const float* isL;
  int H, W, d, block, dir;   // dir: +1 middlebury (q = j - z), -1 paper
  double sigma_eps;
  const int* wc;        // window centre per pixel or kWcNone; nullptr = none
  int64_t ldw;
  int radius;
  double alpha;
  int mode;
  // pipeline outputs (stride ldo)
  int16_t* dout;
  float* cout;
  uint8_t* low;
  int64_t ldo;
  unsigned long long* counters;
  RowBand rows;         // output rows computed / counted
  // padded fp32 staging arrays (prep_staging): R' = R - c and (muR - c,
  // 1/sigma_R | NaN), column margins of `pc` on both sides, row stride ldp
  const float* Rp;
  const float2* Mp;
  int64_t ldp;
  int pc;
  // sweep4 precision guard (one byte per 16 x tile_h tile of the level, row
  // stride flags_ld): sweep4 writes 1 for tiles whose centring amplification
  // is too high and leaves them; sweep2 with fixup = 1 recomputes only those
  const unsigned* tile_flags;
  int64_t flags_ld;
  int tile_h;
  int fixup;
  // fixup list mode: sweep2 walks these job indices (by * fix_nbx + bx)
  const int* fix_list;
  const int* fix_count;
  int fix_nbx;
  // raw outputs (dense H x W): full, window, 3x3-summed winners
  int16_t* fz; float* fc; int16_t* wz; float* wcst; int16_t* nz; float* nc;
  // set by launch_sweep4 (s4_plan): the lanes hold z in [0, s4_ze), the
  // warps' own lanes [0, s4_zm) and a row-split pass the rest; s4_tail:
  // z = d is evaluated once per tile after the sweep
  int s4_ze, s4_zm, s4_tail;
};

cudaError_t launch_sweep(const SweepArgs& a, cudaStream_t s, int* n_launch);
// whether launch_sweep runs sweep4 for these arguments; if so the caller must
// also launch launch_sweep4_fixup (same inputs; may run concurrently)
bool sweep_uses_sweep4(const SweepArgs& a);
cudaError_t launch_sweep4_fixup(const SweepArgs& a, cudaStream_t s);
// job list for launch_sweep4_fixup (after the guard flags, before sweep4)
cudaError_t launch_fixup_list(const unsigned* flags, int64_t flags_ld, int tile_h, int h, int w,
                              RowBand rows, int block, int* list, int* count, cudaStream_t s);
bool sweep_supported_block(int b);
// two-pixels-per-thread variant (sweep2.cu) for b in {3,5,7,9,11}
bool sweep2_supported(int b);
cudaError_t launch_sweep2(const SweepArgs& a, cudaStream_t s);
// disparities-across-lanes variant (sweep4.cu): pipeline mode, b in {5,7,9,11}
bool sweep4_supported(const SweepArgs& a, bool force);
cudaError_t launch_sweep4(const SweepArgs& a, cudaStream_t s);
int sweep4_th();   // output rows per sweep4 tile (the guard's tile height)

// Column margin of the padded staging arrays for search bound d, block b.
inline int staging_margin(int d, int b) { return (d + 16 + b + 40 + 3) / 4 * 4; }
// Rp = fl32(R - c) (replicate-padded columns), Mp = (muR - c, isR > 0 ? isR :
// NaN) inside the image and (0, NaN) in the margins; c: see cR below.
// Rows [y0, y1) only (y1 < 0: all) for row bands.  cR: device pointer to the
// right offset c (pipeline: launch_centre_sample); nullptr: muR at the centre.
cudaError_t launch_prep_staging(const double* R, int64_t ld, const float* muR, const float* isR,
                                int64_t lds, int h, int w, int pc, float* Rp, float2* Mp,
                                int64_t ldp, cudaStream_t s, int y0 = 0, int y1 = -1,
                                const float* cR = nullptr);
// the same from the fp32 level-0 input (identical values: fl32(R - c))
cudaError_t launch_prep_staging(const float* R, int64_t ld, const float* muR, const float* isR,
                                int64_t lds, int h, int w, int pc, float* Rp, float2* Mp,
                                int64_t ldp, cudaStream_t s, int y0 = 0, int y1 = -1,
                                const float* cR = nullptr);
// *out = level-0 right sample at the image centre (fp32 input or fp64 level)
cudaError_t launch_centre_sample(const float* in32, const double* in64, int64_t ld, int h,
                                 int w, float* out, cudaStream_t s);

// ---------------------------------------------------------------- pyramid
cudaError_t launch_f32_to_f64(const float* a, const float* b, int h, int w,
                              int64_t ld_in, double* oa, double* ob,
                              int64_t ld_out, cudaStream_t s);
// two images at once when in1/out1 are non-null
// (output rows [i0, i1) only, i1 < 0: all)
cudaError_t launch_downsample(const double* in0, const double* in1, int h,
                              int w, int64_t ld_in, double* out0, double* out1,
                              int64_t ld_out, cudaStream_t s, int i0 = 0, int i1 = -1);
cudaError_t launch_binomial_smooth(const double* in, int h, int w, int64_t ld_in, double* out,
                                   int64_t ld_out, cudaStream_t s);
// level 1 from the fp32 input, writing the exact fp64 level-0 copy as well
// (rows 2 i0 .. 2 i1 of it)
cudaError_t launch_downsample_f32(const float* in0, const float* in1, int h, int w,
                                  int64_t ld_in, double* out0, double* out1, int64_t ld_out,
                                  double* copy0, double* copy1, int64_t ld_copy,
                                  cudaStream_t s, int i0 = 0, int i1 = -1);

// ---------------------------------------------------------------- stats
// sweep4 precision guard.  sweep4 centres L by one constant per 16 x tile_h
// tile (the L sample at the tile centre, cL) and R by the level constant c
// (the level-0 right sample at the image centre), so the fp32 rounding error
// of its sliding sums, relative to the cost at (p, z), grows with
//   aL(p) x aR(q),  aL = |muL(p) - cL| / sigmaL(p) + 3,  aR = |muR(q) - c| / sigmaR(q) + 3
// for the right pixel q = p -+ z (measured: cost error ~1.1e-7 aL aR).
// The guard bounds it per tile by (max aL over the tile's cost pixels: its
// 16 x tile_h outputs plus the 1-pixel 3x3 border) x (max aR over every right
// pixel those cost pixels meet for z in [0, d]); tiles above
// kSweep4RiskMax get flags[tile] = 1 (zeroed before every run) and sweep4
// leaves them to sweep2's per-pixel centring (launch_sweep4_fixup).
// BASELINE configs stay far below the limit; the reference's smooth
// low-contrast [0, 1] fixtures reach it.
constexpr float kSweep4RiskMax = 200.f;
// sweep4 tile rows (and the guard's tiles) are offset by kTileOff: tile ty
// covers image rows [ty th - kTileOff, (ty + 1) th - kTileOff).  Row bands
// start at multiples of 2^K, so a band's top median halo (its 2 rows above)
// is the last 2 rows of the tile that ends at the band start, not a whole
// extra tile.
constexpr int kTileOff = 2;
__host__ __device__ inline int tile_row(int y, int th) { return (y + kTileOff) / th; }
struct Sweep4Guard {
  const double* L = nullptr;    // level image (cL samples), stride ld
  int64_t ld = 0;
  const float* L32 = nullptr;   // or the fp32 level-0 input, stride ld32
  int64_t ld32 = 0;
  const float* muL = nullptr;   // fp32 statistics, stride lds
  const float* isL = nullptr;
  const float* muR = nullptr;
  const float* isR = nullptr;
  int64_t lds = 0;
  const float* cR = nullptr;    // the right offset c (prep_staging's)
  int h = 0, w = 0, d = 0, dir = 1;
  int tile_h = 0;
  float* colR = nullptr;        // scratch: per (tile row, column) max aR
  unsigned* flags = nullptr;
  int64_t flags_ld = 0;
};
// guard flags of the sweep4 tile rows covering `rows` (two launches)
cudaError_t launch_sweep4_guard(const Sweep4Guard& g, RowBand rows, cudaStream_t s);
// fp32 mean / inverse sigma (0 = degenerate) of the b x b replicate-padded
// window, centred arithmetic in fp64.
cudaError_t launch_stats_f32(const double* img, int h, int w, int64_t ld,
                             int b, double sigma_eps, float* mu, float* is,
                             int64_t lds, cudaStream_t s,
                             int y0 = 0, int y1 = -1);   // rows [y0, y1) (tile-aligned)
// the same from the fp32 level-0 input (b <= 11)
cudaError_t launch_stats_f32(const float* img, int h, int w, int64_t ld, int b, double sigma_eps,
                             float* mu, float* is, int64_t lds, cudaStream_t s, int y0 = 0,
                             int y1 = -1);
// fp64 mean / sigma maps (dense) for the CostEngine API
cudaError_t launch_stats_f64(const double* img, int h, int w, int64_t ld,
                             int b, double* mu, double* sigma, cudaStream_t s);

// ---------------------------------------------------------------- prior
// cubic B-spline prefilter of a coarse cost map into coef
// ((ch+24) x (cw+24), stride ldc); exactly one of c32 / c64 non-null.
cudaError_t launch_bspline_prefilter(const float* c32, const double* c64,
                                     int ch, int cw, int64_t ldcin,
                                     double* coef, int64_t ldc, cudaStream_t s, int r0 = 0,
                                     int r1 = -1);   // padded coefficient rows [r0, r1)
// padded coefficient rows the prior of fine rows `rows` (h fine rows, ch
// coarse rows) reads: the 4 spline taps of every fine row, +-2 rows margin
void prior_coef_rows(int ch, int h, RowBand rows, int* r0, int* r1);
// pipeline prior: window centres from the coarse disparity + spline coef
cudaError_t launch_prior_eval(const int16_t* dcoarse, int64_t ldd, int ch,
                              int cw, const double* coef, int64_t ldc, int h,
                              int w, int d, int radius, double beta, int* wc,
                              int64_t ldw, unsigned long long* counters,
                              RowBand rows, cudaStream_t s);
// stage prior from explicit float64 (d_hat, c_hat) maps (dense h x w)
cudaError_t launch_prior_maps(const double* d_hat, const double* c_hat, int h,
                              int w, int d, int radius, double beta, int* wc,
                              int64_t ldw, unsigned long long* counters,
                              cudaStream_t s);
// upsample_prior stage: d_hat = 2*NN(d), c_hat = clamp(spline)
cudaError_t launch_upsample(const double* dcoarse, int ch, int cw,
                            const double* coef, int64_t ldc, int h, int w,
                            double* d_hat, double* c_hat, cudaStream_t s);

// ---------------------------------------------------------------- median
// pipeline: int16 d, fp32 c, low mask (selection) -> median d, counters
cudaError_t launch_median_pipeline(const int16_t* d, const float* c,
                                   const uint8_t* low, int64_t ld, int h,
                                   int w, double alpha, int16_t* out,
                                   unsigned long long* counters, RowBand rows,
                                   cudaStream_t s);
// stage API: float64 dense maps, NaN-aware
cudaError_t launch_median_f64(const double* d, const double* c, int h, int w,
                              double alpha, double* out,
                              unsigned long long* replaced, cudaStream_t s);

// ---------------------------------------------------------------- evaluate
cudaError_t launch_evaluate(const double* d, const double* gt, const uint8_t* gt_invalid,
                            int64_t n, double scale, const double* taus,
                            unsigned long long* counts, double* abs_sum, cudaStream_t s);

// ---------------------------------------------------------------- engine
struct EngineView {
  const double* L; const double* R; int64_t ld;
  const double* muL; const double* sgL; const double* muR; const double* sgR;
  int H, W, d, block, dir;
  double sigma_eps;
};
cudaError_t launch_engine_plane(const EngineView& e, int z, double* out,
                                cudaStream_t s);
cudaError_t launch_engine_at(const EngineView& e, const int64_t* rows,
                             const int64_t* cols, const int64_t* z, int64_t n,
                             double* out, int* bad, cudaStream_t s);
cudaError_t launch_engine_dsi(const EngineView& e, const int64_t* rows,
                              const int64_t* cols, int64_t n, double* out,
                              int* bad, cudaStream_t s);
// stage combine: select (trusted ? window : full) or refine (low ? nb : in)
cudaError_t launch_combine_select(const int* wc, int h, int w,
                                  const int16_t* fz, const float* fc,
                                  const int16_t* wz, const float* wcst,
                                  double* dout, double* cout, cudaStream_t s);
cudaError_t launch_combine_refine(const double* din, const double* cin, int h,
                                  int w, double alpha, const int16_t* nz,
                                  const float* nc, double* dout, double* cout,
                                  unsigned long long* counters, cudaStream_t s);
cudaError_t launch_low_mask(const double* c, int h, int w, double alpha,
                            int* wc_out, cudaStream_t s);

}  // namespace mshbm
