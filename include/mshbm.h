/*
 * mshbm.h -- C ABI of the B200-native MSHBM disparity engine (libmshbm.so).
 *
 * This is the drop-in boundary for the reference package `pyrstereo`
 * (/root/reference/pkg/src/pyrstereo).  The reference has no FFI of its
 * own: its boundary is the Python function API, so each entry point below
 * names the Python function it replaces (file:line in the reference).  The
 * Python mirror in paper_1901_09593_b200/ binds these with ctypes (see
 * INTEGRATION.md).
 *
 * Conventions
 *  - plain pointers and sizes only; images are row-major with a row stride
 *    ("ld", in elements) >= width;
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *    stream);
 *  - functions taking MSHBM_IO_HOST pointers copy in/out and synchronise;
 *    with MSHBM_IO_DEVICE they are asynchronous on `stream` unless they
 *    return host-side counters (documented per function);
 *  - status codes: 0 ok; MSHBM_ERR_VALUE -> Python ValueError (shapes, z out
 *    of range, non-dyadic upsample, too-deep pyramid), MSHBM_ERR_CONFIG ->
 *    ConfigError (matcher.py:48-84), others -> RuntimeError;
 *  - a context is bound to one device and is not thread-safe.
 */
#ifndef MSHBM_H_
#define MSHBM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSHBM_ABI_VERSION 2

typedef enum {
  MSHBM_OK = 0,
  MSHBM_ERR_VALUE = 1,
  MSHBM_ERR_CONFIG = 2,
  MSHBM_ERR_CUDA = 3,
  MSHBM_ERR_NOMEM = 4,
  MSHBM_ERR_UNSUPPORTED = 5,
  /* codec errors (formats.py exception classes) */
  MSHBM_ERR_DECODE = 10,      /* DecodeError */
  MSHBM_ERR_MALFORMED = 11,   /* MalformedHeaderError */
  MSHBM_ERR_TRUNCATED = 12,   /* TruncatedPayloadError */
  MSHBM_ERR_MAXVAL = 13,      /* UnsupportedMaxvalError */
  MSHBM_ERR_MISSING_KEY = 14  /* MissingKeyError */
} mshbm_status;

enum { MSHBM_SIGN_MIDDLEBURY = 0, MSHBM_SIGN_PAPER = 1 };
enum { MSHBM_IO_DEVICE = 0, MSHBM_IO_HOST = 1 };
/* flags for mshbm_run_pipeline */
enum {
  MSHBM_FLAG_TIMING = 1,   /* fill per-stage milliseconds (read from event-record
                              nodes of the graph; synchronises like a trace) */
  MSHBM_FLAG_NO_GRAPH = 2  /* launch kernels directly instead of a CUDA graph */
};

/* MatchConfig (matcher.py:52-84) plus `radius`, the prior window half-width
 * (the reference hard-codes 1: matcher.py:280,294). levels < 0 = auto. */
typedef struct {
  int32_t d_max;
  int32_t levels;
  int32_t block;
  int32_t radius;
  double alpha;
  double beta;
  double sigma_eps;
  int32_t sign;
  int32_t reserved;
} mshbm_config;

/* LevelTrace (matcher.py:98-153): exact counters + stage milliseconds.
 * ms_build (pyramid construction, PipelineTrace.build_seconds,
 * matcher.py:410-416) and ms_total (whole pipeline on the device) are the
 * same in every level record of one run. */
typedef struct {
  int32_t level, height, width, d_max, block, reserved;
  int64_t trusted;
  int64_t trusted_evals;
  int64_t trusted_window_max;
  int64_t full_search_pixels;
  int64_t selection_evals;
  int64_t refined;
  int64_t refine_evals;
  int64_t median_replaced;
  float ms_upsample, ms_select, ms_refine, ms_median;
  float ms_build, ms_total;
} mshbm_level_trace;

typedef struct mshbm_ctx mshbm_ctx;
typedef struct mshbm_engine mshbm_engine;

/* ---- context ---------------------------------------------------------- */
int mshbm_abi_version(void);
const char* mshbm_status_string(int status);
/* last error message of this context (or of the library if ctx == NULL) */
const char* mshbm_last_error(const mshbm_ctx* ctx);
int mshbm_create(mshbm_ctx** out, int device);
int mshbm_destroy(mshbm_ctx* ctx);
/* count of this library's kernel launches since create (graph replays count
 * every kernel node) -- evidence for bench.py's "gpu_launches". */
int64_t mshbm_launch_count(const mshbm_ctx* ctx);

/* ---- pyramid.py ------------------------------------------------------- */
/* level_d_max / level_block / auto_levels (pyramid.py:84-112) */
int32_t mshbm_level_d_max(int32_t d_max, int32_t k);
int32_t mshbm_level_block(int32_t base_block, int32_t k);
int mshbm_auto_levels(int64_t width, int64_t height, int64_t d_max,
                      int64_t base_block, int32_t* out_levels);
/* Validate `cfg` exactly as MatchConfig.__post_init__ (matcher.py:66-84) and
 * the explicit-K checks of build_pyramid (pyramid.py:139-151) for an HxW pair;
 * writes the resolved K (auto when cfg->levels < 0). */
int mshbm_resolve_levels(const mshbm_config* cfg, int32_t height, int32_t width,
                         int32_t* out_levels);
/* gaussian_downsample (pyramid.py:71-81), float64 device arrays:
 * out is ceil(h/2) x ceil(w/2), row stride ld_out. */
int mshbm_downsample(mshbm_ctx* ctx, const double* in, int32_t h, int32_t w,
                     int64_t ld_in, double* out, int64_t ld_out, void* stream);

/* binomial_smooth (pyramid.py:65-68): the (1,4,6,4,1)/16 filter along axis 0
 * then axis 1 with replicate borders, full resolution (no decimation),
 * float64 device arrays. */
int mshbm_binomial_smooth(mshbm_ctx* ctx, const double* in, int32_t h, int32_t w,
                          int64_t ld_in, double* out, int64_t ld_out, void* stream);

/* ---- whole pipeline (matcher.py:398-466 run_pipeline) ------------------ */
/* left/right: float32 HxW (row stride ld), host or device per `io`.
 * disparity: int16 HxW (stride ld_out), cost: float32 HxW (stride ld_out).
 * trace: array of >= K+1 entries, coarsest level first (may be NULL for a
 * fully asynchronous device call).  Returns K via out_levels (may be NULL). */
int mshbm_run_pipeline(mshbm_ctx* ctx, const float* left, const float* right,
                       int32_t height, int32_t width, int64_t ld,
                       const mshbm_config* cfg, int16_t* disparity, float* cost,
                       int64_t ld_out, mshbm_level_trace* trace,
                       int32_t* out_levels, int32_t io, int32_t flags,
                       void* stream);

/* Row band of run_pipeline for multi-GPU partitioning of one large pair
 * (SURVEY 8e, config C5).  Produces level-0 rows [row_begin, row_end)
 * bit-identical to the whole-image call: the cheap pyramid, statistics and
 * levels >= 2 run on the whole image, levels 0/1 sweep only the band plus
 * exact halos.  row_begin/row_end must be multiples of 2^K (row_end may be
 * H).  disparity/cost receive (row_end - row_begin) rows; trace counters
 * cover only the band's own rows at every level (row_begin>>k .. row_end>>k),
 * so the traces of a partition of bands sum to the whole-image trace
 * (trusted_window_max: take the max). */
int mshbm_run_pipeline_band(mshbm_ctx* ctx, const float* left, const float* right,
                            int32_t height, int32_t width, int64_t ld,
                            const mshbm_config* cfg, int32_t row_begin,
                            int32_t row_end, int16_t* disparity, float* cost,
                            int64_t ld_out, mshbm_level_trace* trace,
                            int32_t* out_levels, int32_t io, int32_t flags,
                            void* stream);

/* Batch of n independent same-shape pairs (config C4): pairs run
 * round-robin on n_streams concurrent CUDA-graph plans (<= 0: 4).  Arrays of
 * n pointers (host or device per `io`); traces: n * (K+1) entries or NULL.
 * Ordered after prior work on `stream`; the call returns with all pairs
 * complete on `stream` (synchronous for host I/O or traces). */
int mshbm_run_batch(mshbm_ctx* ctx, int32_t n_pairs, const float* const* lefts,
                    const float* const* rights, int32_t height, int32_t width,
                    int64_t ld, const mshbm_config* cfg,
                    int16_t* const* disparities, float* const* costs,
                    int64_t ld_out, mshbm_level_trace* traces, int32_t io,
                    int32_t n_streams, void* stream);

/* run_pipeline(..., pyramid=...) with a caller-built pyramid (matcher.py:
 * 410-416): n_levels float64 device levels, level k has dims heights[k] x
 * widths[k] (dyadic), stride lds[k], search bound d_maxs[k], block blocks[k]. */
int mshbm_run_pyramid(mshbm_ctx* ctx, int32_t n_levels,
                      const double* const* lefts, const double* const* rights,
                      const int32_t* heights, const int32_t* widths,
                      const int64_t* lds, const int32_t* d_maxs,
                      const int32_t* blocks, const mshbm_config* cfg,
                      int16_t* disparity, float* cost, int64_t ld_out,
                      mshbm_level_trace* trace, void* stream);

/* ---- CostEngine (zncc.py:144-307) ------------------------------------- */
/* Device-resident level: copies float64 device images (HxW, stride ld). */
int mshbm_engine_create(mshbm_ctx* ctx, const double* left, const double* right,
                        int32_t height, int32_t width, int64_t ld, int32_t block,
                        int32_t d_max, double sigma_eps, int32_t sign,
                        mshbm_engine** out);
int mshbm_engine_destroy(mshbm_engine* e);
/* box mean / sigma maps of both images (zncc.py:185-189), float64 HxW dense */
int mshbm_engine_stats(mshbm_engine* e, double* mean_l, double* sigma_l,
                       double* mean_r, double* sigma_r, void* stream);
/* CostEngine.plane (zncc.py:202-231): costs of every pixel at z, HxW f64 */
int mshbm_engine_plane(mshbm_engine* e, int32_t z, double* out, void* stream);
/* CostEngine.at (zncc.py:251-269): n (row, col, z) triples -> out[n] f64.
 * z outside [0, d_max] -> MSHBM_ERR_VALUE (checked on device, synchronous) */
int mshbm_engine_at(mshbm_engine* e, const int64_t* rows, const int64_t* cols,
                    const int64_t* z, int64_t n, double* out, void* stream);
/* CostEngine.dsi_rows (zncc.py:289-302): out is n x (d_max+1) f64 */
int mshbm_engine_dsi_rows(mshbm_engine* e, const int64_t* rows,
                          const int64_t* cols, int64_t n, double* out,
                          void* stream);
/* match_coarsest (matcher.py:184-193): fused full-range ZNCC + WTA.
 * disparity/cost: HxW f64 dense. */
int mshbm_match_coarsest(mshbm_engine* e, double* disparity, double* cost,
                         void* stream);
/* select_with_prior (matcher.py:263-320) with window +-radius.
 * stats[5] = {trusted, trusted_evals, window_max, full_search_pixels, evals}
 * (host memory; the call synchronises). */
int mshbm_select_with_prior(mshbm_engine* e, const double* d_hat,
                            const double* c_hat, double beta, int32_t radius,
                            double* disparity, double* cost, int64_t* stats,
                            void* stream);
/* refine_level (matcher.py:196-233). evals (host) = |dilate(low)|*(d+1)
 * or 0; the call synchronises. */
int mshbm_refine_level(mshbm_engine* e, const double* disparity,
                       const double* cost, double alpha, double* out_disparity,
                       double* out_cost, int64_t* evals, void* stream);

/* ---- stage kernels without an engine ---------------------------------- */
/* selective_median (matcher.py:323-359), f64 HxW dense; replaced (host,
 * may be NULL) = number of changed pixels (NaN==NaN counts unchanged). */
int mshbm_selective_median(mshbm_ctx* ctx, const double* disparity,
                           const double* cost, int32_t height, int32_t width,
                           double alpha, double* out, int64_t* replaced,
                           void* stream);
/* upsample_prior (matcher.py:236-260): coarse ch x cw -> h x w, f64 dense */
int mshbm_upsample_prior(mshbm_ctx* ctx, const double* d_coarse,
                         const double* c_coarse, int32_t ch, int32_t cw,
                         int32_t h, int32_t w, double* d_hat, double* c_hat,
                         void* stream);

/* ---- scoring (SURVEY 8f "next": device-side evaluate) ------------------ */
/* evaluate (evaluation.py:77-109) on device arrays of n pixels: disparity
 * (f64, NaN = invalid), gt_values (f64), gt_invalid (u8), scale > 0,
 * taus[3] = bad thresholds (1, 2, 4).  Host outputs: counts[6] = {evaluated,
 * bad_tau0, bad_tau1, bad_tau2, gt_invalid, output_invalid}, abs_err_sum =
 * sum over evaluated pixels of |disparity*scale - gt|.  Synchronises. */
int mshbm_evaluate(mshbm_ctx* ctx, const double* disparity, const double* gt_values,
                   const uint8_t* gt_invalid, int64_t n, double scale,
                   const double* taus, int64_t* counts, double* abs_err_sum,
                   void* stream);

/* ---- wire formats (formats.py:123-278) ---------------- *
 * Host-side codecs over in-memory file bytes; errors set mshbm_last_error(NULL)
 * with the reference's messages and return the MSHBM_ERR_* decode codes. */
typedef struct {
  int32_t width, height, maxval, channels; /* channels 1 (P2/P5) or 3 (P3/P6) */
  int32_t ascii;                           /* P2/P3 */
  int32_t itemsize;                        /* binary bytes per sample (maxval > 255: 2, BE) */
  int64_t payload_offset;                  /* first payload byte (binary) / token (ASCII) */
} mshbm_pnm_header;

typedef struct {
  int32_t width, height;
  double scale;                            /* < 0 little endian, > 0 big endian */
  int64_t payload_offset;
} mshbm_pfm_header;

/* read_pnm header checks (formats.py:123-175) */
int mshbm_pnm_parse(const uint8_t* buf, int64_t len, mshbm_pnm_header* hdr);
/* read_pnm samples -> grayscale in [0, 1], fp64 host (formats.py:150-190) */
int mshbm_pnm_decode(const uint8_t* buf, int64_t len, const mshbm_pnm_header* hdr,
                     double* gray, int64_t ld);
/* binary PNM payload -> fp32 grayscale on the device (raw samples cross
 * PCIe); synchronises `stream` to report out-of-range samples */
int mshbm_pnm_upload(const uint8_t* buf, int64_t len, const mshbm_pnm_header* hdr,
                     float* d_gray, int64_t ld, void* stream);
/* read_pfm (formats.py:193-232): header, then rows flipped to top-down,
 * non-finite samples -> NaN values and invalid = 1 */
int mshbm_pfm_parse(const uint8_t* buf, int64_t len, mshbm_pfm_header* hdr);
int mshbm_pfm_decode(const uint8_t* buf, int64_t len, const mshbm_pfm_header* hdr,
                     double* values, uint8_t* invalid, int64_t ld);
/* write_pfm / write_pgm (formats.py:235-278): return the encoded size in
 * bytes (writing only when cap suffices), or -MSHBM_ERR_VALUE */
int64_t mshbm_pfm_encode(const double* values, int32_t h, int32_t w, int64_t ld, double scale,
                         uint8_t* out, int64_t cap);
int64_t mshbm_pgm_encode(const double* values, int32_t h, int32_t w, int64_t ld,
                         int32_t maxval, double scale_max, uint8_t* out, int64_t cap);

/* ---- diagnostics ------------------------------------------------------- */
/* FP32 FFMA throughput of `device` (8 CTAs/SM x 256 threads, 8 independent
 * FMA chains per thread, `iters` x 128 FMAs): the roofline denominator of
 * the ZNCC sweep (not part of the reference interface). */
int mshbm_probe_fp32_peak(int device, int iters, double* tflops, double* ms);
/* FP64 DFMA throughput, same shape (diagnostics). */
int mshbm_probe_fp64_peak(int device, int iters, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* MSHBM_H_ */
