/* CPU oracle for the MSHBM disparity hot path, plain C + OpenMP.
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke(), bench.py's CPU
 * baseline leg and tools/make_golden.py load it; the product package never
 * does.
 *
 * A float64 restatement of the reference `run_pipeline`
 * (/root/reference/pkg/src/pyrstereo/matcher.py:398-466) with the prior
 * window generalised to +-radius (matcher.py:280,294 hard-code 1; radius=1
 * is the reference).  It exists because the reference (and the numpy
 * restatement in mshbm_oracle.py) materialise S x (d+1) float64 DSI rows
 * (zncc.py:289-302): full-size C5 would need ~0.5 TB and ~4 h.  Here every
 * level is swept row by row over a 3-row ring of dense DSI rows, so memory
 * is O(threads * 3 * (d+1) * W) and the rows are computed once.
 *
 * Arithmetic per stage (all float64, the reference's formulas; only the
 * summation order of the window sums differs, ~1e-15 relative):
 *   pyramid      pyramid.py:65-81   correlate1d([1,4,6,4,1]/16, 'nearest')
 *                                   axis 0 then axis 1, keep [::2, ::2]
 *                                   (scipy's symmetric-kernel accumulation)
 *   stats        zncc.py:175-189    uniform_filter(mode='nearest') as scipy's
 *                                   running-sum uniform_filter1d, axis 0 then 1;
 *                                   sigma = sqrt(max(E[x^2]-mu^2, 0)); ok = sigma >= eps
 *   ZNCC         zncc.py:271-287    cross = sum of L_pad*R_pad over the bxb window,
 *                                   cov = cross/b^2 - muL*muR, rho = clip(cov/(sL*sR)),
 *                                   -1 when !okL, !okR or the right centre leaves
 *                                   the image.  Evaluated as column sums V(c) of
 *                                   the b row products, then sum_t V(j+t).
 *   coarsest     matcher.py:184-193 first argmax over z = 0..d
 *   upsample     matcher.py:236-260 2x NN disparity; scipy map_coordinates(order=3,
 *                                   mode='nearest'): 12-sample edge prepad, cubic
 *                                   B-spline prefilter (pole sqrt(3)-2, 'reflect'
 *                                   causal init) per axis, 4x4 tap sampling, clamp
 *   select       matcher.py:263-320 trusted = c_hat > beta & finite & window meets
 *                                   [0, d]; ascending window, strict '>' vs -2;
 *                                   untrusted: first argmax of the full row
 *   refine       matcher.py:196-233 low = C <= alpha; for low px the clipped 3x3
 *                                   neighbour sum (di outer, dj inner), first
 *                                   argmax, C = sum[best]/members
 *   median       matcher.py:323-359 lower median of the 5x5 neighbours with
 *                                   C > alpha and finite d (cost padded -2)
 *   counters     matcher.py:372-466 closed forms
 *
 * Parity: pinned against the real reference's outputs (tests/golden/ fixtures,
 * tools/make_golden.py) in tests/test_oracle_c.py.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EVALUE 1
#define ORC_ENOMEM 2

enum { T_LEVEL, T_HEIGHT, T_WIDTH, T_DMAX, T_BLOCK, T_TRUSTED, T_TRUSTED_EVALS,
       T_WINDOW_MAX, T_FULL, T_SELECTION_EVALS, T_REFINED, T_REFINE_EVALS,
       T_MEDIAN_REPLACED, T_NCOLS };

static int level_d_max(int d, int k) { int v = d >> k; return v < 1 ? 1 : v; }   /* pyramid.py:84-86 */
static int level_block(int b, int k) {                                          /* pyramid.py:89-94 */
    int v = b >> k;
    if (v % 2 == 0) v -= 1;
    return v < 3 ? 3 : v;
}

int mshbm_oracle_auto_levels(int width, int height, int d_max, int base_block) {
    /* pyramid.py:97-112 */
    if ((width < height ? width : height) <= 0 || d_max < 1 || base_block < 1) return -1;
    int k = 0, m = width < height ? width : height;
    while ((double)m / (double)(1 << (k + 1)) >= 4.0 * base_block && (d_max >> (k + 1)) >= 2) k++;
    return k;
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* gaussian_downsample (pyramid.py:65-81): scipy correlate1d with a symmetric
 * 5-tap kernel accumulates x0*w0 + (x-2 + x+2)*w2 + (x-1 + x+1)*w1. */
static void downsample(const double* in, int h, int w, double* out) {
    const double w0 = 6.0 / 16.0, w1 = 4.0 / 16.0, w2 = 1.0 / 16.0;
    int oh = (h + 1) / 2, ow = (w + 1) / 2;
    #pragma omp parallel
    {
        double* v = (double*)malloc(sizeof(double) * (size_t)w);
        #pragma omp for schedule(static)
        for (int oi = 0; oi < oh; ++oi) {
            int i = 2 * oi;
            const double* r0 = in + (size_t)clampi(i - 2, 0, h - 1) * w;
            const double* r1 = in + (size_t)clampi(i - 1, 0, h - 1) * w;
            const double* r2 = in + (size_t)i * w;
            const double* r3 = in + (size_t)clampi(i + 1, 0, h - 1) * w;
            const double* r4 = in + (size_t)clampi(i + 2, 0, h - 1) * w;
            for (int j = 0; j < w; ++j) {
                double t = r2[j] * w0;
                t += (r0[j] + r4[j]) * w2;
                t += (r1[j] + r3[j]) * w1;
                v[j] = t;
            }
            for (int oj = 0; oj < ow; ++oj) {
                int j = 2 * oj;
                double t = v[j] * w0;
                t += (v[clampi(j - 2, 0, w - 1)] + v[clampi(j + 2, 0, w - 1)]) * w2;
                t += (v[clampi(j - 1, 0, w - 1)] + v[clampi(j + 1, 0, w - 1)]) * w1;
                out[(size_t)oi * ow + oj] = t;
            }
        }
        free(v);
    }
}

/* scipy uniform_filter1d(mode='nearest') on one extended line: running sum. */
static void uniform_line(const double* ext, int n, int size, double* out, ptrdiff_t ostride) {
    double tmp = 0.0;
    for (int k = 0; k < size; ++k) tmp += ext[k];
    tmp /= (double)size;
    out[0] = tmp;
    for (int k = 1; k < n; ++k) {
        tmp += (ext[k + size - 1] - ext[k - 1]) / (double)size;
        out[(ptrdiff_t)k * ostride] = tmp;
    }
}

/* uniform_filter(img (optionally squared), b, mode='nearest'): axis 0 then 1. */
static void box_mean(const double* img, int h, int w, int b, int square, double* out) {
    int half = b / 2;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)h * w);
    #pragma omp parallel
    {
        int mx = (h > w ? h : w) + b;
        double* ext = (double*)malloc(sizeof(double) * (size_t)mx);
        double* col = (double*)malloc(sizeof(double) * (size_t)mx);
        #pragma omp for schedule(static)
        for (int j = 0; j < w; ++j) {             /* axis 0 (columns) */
            for (int k = 0; k < h + 2 * half; ++k) {
                double v = img[(size_t)clampi(k - half, 0, h - 1) * w + j];
                ext[k] = square ? v * v : v;
            }
            uniform_line(ext, h, b, col, 1);
            for (int i = 0; i < h; ++i) tmp[(size_t)i * w + j] = col[i];
        }
        #pragma omp for schedule(static)
        for (int i = 0; i < h; ++i) {             /* axis 1 (rows) */
            for (int k = 0; k < w + 2 * half; ++k) ext[k] = tmp[(size_t)i * w + clampi(k - half, 0, w - 1)];
            uniform_line(ext, w, b, out + (size_t)i * w, 1);
        }
        free(ext);
        free(col);
    }
    free(tmp);
}

typedef struct {
    int h, w, b, half, d, sign;        /* sign 0 = middlebury (q = j - z), 1 = paper (q = j + z) */
    int pw;                            /* padded width w + 2*half */
    double *lp, *rp;                   /* edge-padded images (h+2half) x pw */
    double *mul, *sl, *mur, *sr;       /* stats */
    unsigned char *okl, *okr;
} Engine;

static void engine_free(Engine* e) {
    free(e->lp); free(e->rp); free(e->mul); free(e->sl); free(e->mur); free(e->sr);
    free(e->okl); free(e->okr);
}

static int engine_init(Engine* e, const double* L, const double* R, int h, int w, int b, int d,
                       double eps, int sign) {
    memset(e, 0, sizeof(*e));
    e->h = h; e->w = w; e->b = b; e->half = b / 2; e->d = d; e->sign = sign;
    e->pw = w + 2 * e->half;
    size_t ph = (size_t)h + 2 * e->half, n = (size_t)h * w;
    e->lp = (double*)malloc(sizeof(double) * ph * e->pw);
    e->rp = (double*)malloc(sizeof(double) * ph * e->pw);
    e->mul = (double*)malloc(sizeof(double) * n);
    e->sl = (double*)malloc(sizeof(double) * n);
    e->mur = (double*)malloc(sizeof(double) * n);
    e->sr = (double*)malloc(sizeof(double) * n);
    e->okl = (unsigned char*)malloc(n);
    e->okr = (unsigned char*)malloc(n);
    double* sq = (double*)malloc(sizeof(double) * n);
    if (!e->lp || !e->rp || !e->mul || !e->sl || !e->mur || !e->sr || !e->okl || !e->okr || !sq) {
        free(sq); engine_free(e); return ORC_ENOMEM;
    }
    #pragma omp parallel for schedule(static)
    for (long long pi = 0; pi < (long long)ph; ++pi) {   /* np.pad(img, half, 'edge') */
        int si = clampi((int)pi - e->half, 0, h - 1);
        for (int pj = 0; pj < e->pw; ++pj) {
            int sj = clampi(pj - e->half, 0, w - 1);
            e->lp[(size_t)pi * e->pw + pj] = L[(size_t)si * w + sj];
            e->rp[(size_t)pi * e->pw + pj] = R[(size_t)si * w + sj];
        }
    }
    for (int side = 0; side < 2; ++side) {                 /* zncc.py:185-189 */
        const double* img = side ? R : L;
        double* mu = side ? e->mur : e->mul;
        double* sg = side ? e->sr : e->sl;
        unsigned char* ok = side ? e->okr : e->okl;
        box_mean(img, h, w, b, 0, mu);
        box_mean(img, h, w, b, 1, sq);
        #pragma omp parallel for schedule(static)
        for (long long p = 0; p < (long long)n; ++p) {
            double v = sq[p] - mu[p] * mu[p];
            sg[p] = sqrt(v > 0.0 ? v : 0.0);
            ok[p] = sg[p] >= eps;
        }
    }
    free(sq);
    return ORC_OK;
}

/* Dense DSI row i: out[z*w + j] = rho(i, j, z) for z = 0..d (zncc.py:271-287).
 * vbuf: scratch of 2 * (pw + 2d + 8) doubles. */
static void dsi_row(const Engine* e, int i, double* out, double* vbuf) {
    const int w = e->w, b = e->b, pw = e->pw, d = e->d;
    const double area = (double)(b * b);
    const double* mul = e->mul + (size_t)i * w;
    const double* sl = e->sl + (size_t)i * w;
    const double* mur = e->mur + (size_t)i * w;
    const double* sr = e->sr + (size_t)i * w;
    const unsigned char* okl = e->okl + (size_t)i * w;
    const unsigned char* okr = e->okr + (size_t)i * w;
    for (int z = 0; z <= d; ++z) {
        double* o = out + (size_t)z * w;
        /* valid output columns: right centre q in [0, w-1] */
        int j0, j1;
        if (e->sign == 0) { j0 = z; j1 = w; } else { j0 = 0; j1 = w - z; }
        for (int j = 0; j < w; ++j) o[j] = -1.0;
        if (j0 >= j1) continue;
        /* V(c) over padded L columns c in [j0, j1 + b - 1): sum_p L_pad*R_pad */
        int c0 = j0, c1 = j1 + b - 1;
        int off = e->sign == 0 ? -z : z;
        for (int c = c0; c < c1; ++c) vbuf[c] = 0.0;
        for (int p = 0; p < b; ++p) {
            const double* lr = e->lp + (size_t)(i + p) * pw;
            const double* rr = e->rp + (size_t)(i + p) * pw + off;
            for (int c = c0; c < c1; ++c) vbuf[c] += lr[c] * rr[c];
        }
        /* cross(j) = sum_t V(j + t), accumulated t-outer (vectorises over j) */
        double* cr = vbuf + pw + 2 * d + 8;
        for (int j = j0; j < j1; ++j) cr[j] = vbuf[j];
        for (int t = 1; t < b; ++t)
            for (int j = j0; j < j1; ++j) cr[j] += vbuf[j + t];
        for (int j = j0; j < j1; ++j) {
            int q = j + off;
            double cov = cr[j] / area - mul[j] * mur[q];
            double den = sl[j] * sr[q];
            double r = (okl[j] & okr[q]) ? cov / den : -1.0;
            r = r < -1.0 ? -1.0 : r;
            o[j] = r > 1.0 ? 1.0 : r;
        }
    }
}

/* ---------------------------------------------------------------- B-spline */
#define NPAD 12

static void spline_filter_line(double* c, int n, ptrdiff_t s) {
    /* scipy spline_filter1d(order=3) on one line (mshbm_oracle.py
     * _spline_filter_axis, pinned to scipy 1.18.1). */
    const double z = sqrt(3.0) - 2.0;
    const double gain = (1.0 - z) * (1.0 - 1.0 / z);
    for (int i = 0; i < n; ++i) c[i * s] *= gain;
    if (n <= 1) return;
    double zn = pow(z, (double)n);
    double c0 = c[0];
    double acc = c[0] + zn * c[(n - 1) * s];
    double zi = z;
    for (int i = 1; i < n; ++i) {
        acc = acc + zi * (c[i * s] + zn * c[(n - 1 - i) * s]);
        zi *= z;
        if (zi == 0.0) break;
    }
    c[0] = acc * (z / (1.0 - zn * zn)) + c0;
    for (int i = 1; i < n; ++i) c[i * s] += z * c[(i - 1) * s];
    c[(n - 1) * s] *= z / (z - 1.0);
    for (int i = n - 2; i >= 0; --i) c[i * s] = z * (c[(i + 1) * s] - c[i * s]);
}

static void bspline_weights(double t, double wt[4]) {
    wt[0] = (1.0 - t) * (1.0 - t) * (1.0 - t) / 6.0;
    wt[1] = (4.0 - 6.0 * t * t + 3.0 * t * t * t) / 6.0;
    wt[2] = (1.0 + 3.0 * t + 3.0 * t * t - 3.0 * t * t * t) / 6.0;
    wt[3] = t * t * t / 6.0;
}

/* upsample_prior (matcher.py:236-260) */
static int upsample_prior(const double* dc, const double* cc, int ch, int cw, int h, int w,
                          double* dh, double* chat) {
    if (ch != (h + 1) / 2 || cw != (w + 1) / 2) return ORC_EVALUE;
    int ph = ch + 2 * NPAD, pw = cw + 2 * NPAD;
    double* coef = (double*)malloc(sizeof(double) * (size_t)ph * pw);
    if (!coef) return ORC_ENOMEM;
    for (int i = 0; i < ph; ++i)
        for (int j = 0; j < pw; ++j)
            coef[(size_t)i * pw + j] = cc[(size_t)clampi(i - NPAD, 0, ch - 1) * cw + clampi(j - NPAD, 0, cw - 1)];
    #pragma omp parallel for schedule(static)
    for (int j = 0; j < pw; ++j) spline_filter_line(coef + j, ph, pw);      /* axis 0 */
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < ph; ++i) spline_filter_line(coef + (size_t)i * pw, pw, 1);   /* axis 1 */
    double sy = (double)ch / (double)h, sx = (double)cw / (double)w;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < h; ++i) {
        double y = ((double)i + 0.5) * sy - 0.5 + NPAD;
        double fy = floor(y), wy[4];
        bspline_weights(y - fy, wy);
        int iy = (int)fy - 1;
        for (int j = 0; j < w; ++j) {
            double x = ((double)j + 0.5) * sx - 0.5 + NPAD;
            double fx = floor(x), wx[4];
            bspline_weights(x - fx, wx);
            int ix = (int)fx - 1;
            double out = 0.0;
            for (int a = 0; a < 4; ++a) {
                int ry = clampi(iy + a, 0, ph - 1);
                double row = 0.0;
                for (int t = 0; t < 4; ++t) row = row + wx[t] * coef[(size_t)ry * pw + clampi(ix + t, 0, pw - 1)];
                out = out + wy[a] * row;
            }
            chat[(size_t)i * w + j] = out < -1.0 ? -1.0 : (out > 1.0 ? 1.0 : out);
            dh[(size_t)i * w + j] = 2.0 * dc[(size_t)(i / 2) * cw + (j / 2)];
        }
    }
    free(coef);
    return ORC_OK;
}

/* selection of one row from its dense DSI row (matcher.py:263-320).  z
 * runs in the outer loop (the row is plane-major); bz/bc: scratch of w. */
static void select_row(const Engine* e, const double* row, int i, const int* wsz,
                       const double* dhat, int radius, double* dsel, double* csel,
                       int* bz, double* bc) {
    const int w = e->w, d = e->d;
    const int* ws = wsz + (size_t)i * w;
    const double* dh = dhat ? dhat + (size_t)i * w : NULL;
    for (int j = 0; j < w; ++j) {
        bz[j] = 0;
        bc[j] = ws[j] < 0 ? row[j] : -2.0;        /* full search: z = 0 is the first max */
    }
    for (int z = 0; z <= d; ++z) {
        const double* rz = row + (size_t)z * w;
        for (int j = 0; j < w; ++j) {
            if (ws[j] < 0) {
                if (z > 0 && rz[j] > bc[j]) { bc[j] = rz[j]; bz[j] = z; }
            } else {                               /* ascending window, strict > vs -2 */
                long long ctr = (long long)dh[j];
                if (z >= ctr - radius && z <= ctr + radius && rz[j] > bc[j]) { bc[j] = rz[j]; bz[j] = z; }
            }
        }
    }
    for (int j = 0; j < w; ++j) {
        dsel[(size_t)i * w + j] = (double)bz[j];
        csel[(size_t)i * w + j] = bc[j];
    }
}

/* refinement of row i's low pixels (matcher.py:196-233); the ring holds
 * the DSI rows i-1, i, i+1 at slots (row % 3).  The clipped 3x3 sum of each
 * pixel accumulates in the reference's order (di outer, dj inner); z runs
 * in the outer loop.  bz/bs/acc: scratch of w. */
static void refine_row(const Engine* e, const double* ring, size_t rowsz, int i, double alpha,
                       const double* dsel, const double* csel, double* dref, double* cref,
                       int* bz, double* bs, double* acc) {
    const int h = e->h, w = e->w, d = e->d;
    const double* cs = csel + (size_t)i * w;
    int any = 0;
    for (int j = 0; j < w; ++j) {
        dref[(size_t)i * w + j] = dsel[(size_t)i * w + j];
        cref[(size_t)i * w + j] = cs[j];
        any |= cs[j] <= alpha;
    }
    if (!any) return;
    for (int z = 0; z <= d; ++z) {
        for (int j = 0; j < w; ++j) acc[j] = 0.0;
        for (int di = -1; di <= 1; ++di) {
            int qi = i + di;
            if (qi < 0 || qi >= h) continue;
            const double* rz = ring + (size_t)(qi % 3) * rowsz + (size_t)z * w;
            acc[0] += rz[0];                              /* j = 0: dj = 0, +1 */
            if (w > 1) acc[0] += rz[1];
            for (int j = 1; j < w - 1; ++j) {
                double t = acc[j] + rz[j - 1];
                t += rz[j];
                acc[j] = t + rz[j + 1];
            }
            if (w > 1) { acc[w - 1] += rz[w - 2]; acc[w - 1] += rz[w - 1]; }
        }
        for (int j = 0; j < w; ++j)
            if (z == 0 || acc[j] > bs[j]) { bs[j] = acc[j]; bz[j] = z; }
    }
    for (int j = 0; j < w; ++j) {
        if (!(cs[j] <= alpha)) continue;
        int rows_in = 1 + (i > 0) + (i < h - 1);
        int cols_in = 1 + (j > 0) + (j < w - 1);
        dref[(size_t)i * w + j] = (double)bz[j];
        cref[(size_t)i * w + j] = bs[j] / (double)(rows_in * cols_in);
    }
}

/* ------------------------------------------------------------ one level */
/* select (or full search when dhat == NULL), refine and median for one
 * level.  Writes d_out (post-median), c_out (refined cost), counters. */
static int process_level(const Engine* e, const double* dhat, const double* chat, double alpha,
                         double beta, int radius, double* d_out, double* c_out, int64_t* tr) {
    const int h = e->h, w = e->w, d = e->d;
    const size_t n = (size_t)h * w;
    double* dsel = (double*)malloc(sizeof(double) * n);
    double* csel = (double*)malloc(sizeof(double) * n);
    double* dref = (double*)malloc(sizeof(double) * n);
    int* wsz = (int*)calloc(n, sizeof(int));                 /* window size, -1 = untrusted */
    if (!dsel || !csel || !dref || !wsz) { free(dsel); free(csel); free(dref); free(wsz); return ORC_ENOMEM; }
    /* trusted mask + window sizes (matcher.py:278-281) */
    #pragma omp parallel for schedule(static)
    for (long long p = 0; p < (long long)n; ++p) {
        if (!dhat) { wsz[p] = -1; continue; }
        double dv = dhat[p];
        int fin = isfinite(dv);
        long long ctr = fin ? (long long)dv : 0;          /* astype(np.intp) truncates */
        int ok = fin && ctr + radius >= 0 && ctr - radius <= d && chat[p] > beta;
        if (!ok) { wsz[p] = -1; continue; }
        long long lo = ctr - radius < 0 ? 0 : ctr - radius;
        long long hi = ctr + radius > d ? d : ctr + radius;
        wsz[p] = (int)(hi - lo + 1);
    }
    /* selection and refinement, row bands over a 3-row DSI ring */
    const int band = 16;
    const int nb = (h + band - 1) / band;
    int err = 0;
    #pragma omp parallel
    {
        size_t rowsz = (size_t)(d + 1) * w;
        double* ring = (double*)malloc(sizeof(double) * rowsz * 3);
        double* vbuf = (double*)malloc(sizeof(double) * (size_t)(2 * (e->pw + 2 * d + 8)));
        int* sbz = (int*)malloc(sizeof(int) * (size_t)w);
        double* sbc = (double*)malloc(sizeof(double) * (size_t)w);
        double* sacc = (double*)malloc(sizeof(double) * (size_t)w);
        int have[3] = {-1, -1, -1};
        if (!ring || !vbuf || !sbz || !sbc || !sacc) {
            #pragma omp atomic write
            err = ORC_ENOMEM;
        }
        #pragma omp for schedule(dynamic, 1)
        for (int bi = 0; bi < nb; ++bi) {
            if (err) continue;
            int r0 = bi * band, r1 = r0 + band < h ? r0 + band : h;
            /* rows r0-1 .. r1 stream through the ring; row t is refined as
             * soon as row t+1 (its lower 3x3 neighbour) is in the ring */
            int lo = r0 > 0 ? r0 - 1 : 0, hi = r1 < h ? r1 : h - 1;
            for (int i = lo; i <= hi; ++i) {
                int slot = i % 3;
                if (have[slot] != i) { dsi_row(e, i, ring + slot * rowsz, vbuf); have[slot] = i; }
                if (i >= r0 && i < r1)
                    select_row(e, ring + slot * rowsz, i, wsz, dhat, radius, dsel, csel, sbz, sbc);
                if (i - 1 >= r0 && i - 1 < r1)
                    refine_row(e, ring, rowsz, i - 1, alpha, dsel, csel, dref, c_out, sbz, sbc, sacc);
            }
            if (hi == r1 - 1)
                refine_row(e, ring, rowsz, r1 - 1, alpha, dsel, csel, dref, c_out, sbz, sbc, sacc);
        }
        free(ring); free(vbuf); free(sbz); free(sbc); free(sacc);
    }
    if (err) { free(dsel); free(csel); free(dref); free(wsz); return err; }
    /* counters */
    int64_t trusted = 0, tevals = 0, wmax = 0, refined = 0, needed = 0, replaced = 0;
    #pragma omp parallel for reduction(+:trusted, tevals, refined, needed) reduction(max:wmax) schedule(static)
    for (long long p = 0; p < (long long)n; ++p) {
        if (wsz[p] >= 0) { trusted++; tevals += wsz[p]; if (wsz[p] > wmax) wmax = wsz[p]; }
        if (csel[p] <= alpha) refined++;
        int i = (int)(p / w), j = (int)(p % w), nd = 0;
        for (int di = -1; di <= 1 && !nd; ++di)
            for (int dj = -1; dj <= 1; ++dj) {
                int qi = i + di, qj = j + dj;
                if (qi >= 0 && qi < h && qj >= 0 && qj < w && csel[(size_t)qi * w + qj] <= alpha) { nd = 1; break; }
            }
        needed += nd;
    }
    /* selective median on the refined maps (matcher.py:323-359) */
    #pragma omp parallel for reduction(+:replaced) schedule(static)
    for (int i = 0; i < h; ++i) {
        double pool[25];
        for (int j = 0; j < w; ++j) {
            size_t p = (size_t)i * w + j;
            double v = dref[p];
            if (c_out[p] <= alpha) {
                int m = 0;
                for (int di = -2; di <= 2; ++di)
                    for (int dj = -2; dj <= 2; ++dj) {
                        int qi = i + di, qj = j + dj;
                        if (qi < 0 || qi >= h || qj < 0 || qj >= w) continue;   /* padded -2 */
                        size_t q = (size_t)qi * w + qj;
                        if (c_out[q] > alpha && isfinite(dref[q])) {
                            double x = dref[q];
                            int k = m++;
                            while (k > 0 && pool[k - 1] > x) { pool[k] = pool[k - 1]; --k; }
                            pool[k] = x;
                        }
                    }
                if (m > 0) v = pool[(m - 1) / 2];
            }
            d_out[p] = v;
            int both_nan = isnan(v) && isnan(dref[p]);
            if (!both_nan && v != dref[p]) replaced++;
        }
    }
    tr[T_HEIGHT] = h; tr[T_WIDTH] = w; tr[T_DMAX] = d; tr[T_BLOCK] = e->b;
    if (dhat) {
        tr[T_TRUSTED] = trusted; tr[T_TRUSTED_EVALS] = tevals; tr[T_WINDOW_MAX] = wmax;
        tr[T_FULL] = (int64_t)n - trusted;
        tr[T_SELECTION_EVALS] = tevals + ((int64_t)n - trusted) * (d + 1);
    } else {
        tr[T_TRUSTED] = 0; tr[T_TRUSTED_EVALS] = 0; tr[T_WINDOW_MAX] = 0;
        tr[T_FULL] = (int64_t)n; tr[T_SELECTION_EVALS] = (int64_t)n * (d + 1);
    }
    tr[T_REFINED] = refined;
    tr[T_REFINE_EVALS] = refined ? needed * (d + 1) : 0;
    tr[T_MEDIAN_REPLACED] = replaced;
    free(dsel); free(csel); free(dref); free(wsz);
    return ORC_OK;
}

int mshbm_oracle_trace_cols(void) { return T_NCOLS; }

/* run_pipeline (matcher.py:398-466) with radius r.  levels < 0 = auto.
 * trace: (levels+1) x T_NCOLS int64, coarsest level first (the golden
 * `counts` layout).  level_d/level_c (optional): every level's final
 * disparity and (refined) cost map, levels 0..K concatenated (teacher-forced
 * stage parity).  Returns 0, or 1 for a ValueError, 2 for out of memory. */
int mshbm_oracle_run_pipeline(const double* left, const double* right, int height, int width,
                              int d_max, int levels, int block, int radius, double alpha,
                              double beta, double sigma_eps, int sign, int threads,
                              double* d_out, double* c_out, int64_t* trace, int* levels_out,
                              double* level_d, double* level_c) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    if (height < 1 || width < 1 || d_max < 1 || block < 3 || block % 2 == 0 || radius < 0) return ORC_EVALUE;
    if (levels < 0) levels = mshbm_oracle_auto_levels(width, height, d_max, block);
    if (levels > 0) {                                    /* pyramid.py:139-151 */
        int hh = height, ww = width;
        for (int k = 0; k < levels; ++k) { hh = (hh + 1) / 2; ww = (ww + 1) / 2; }
        if ((hh < ww ? hh : ww) < 2 * level_block(block, levels)) return ORC_EVALUE;
        if ((d_max >> levels) < 2) return ORC_EVALUE;
    }
    if (levels_out) *levels_out = levels;
    int K = levels;
    double** L = (double**)calloc(K + 1, sizeof(double*));
    double** R = (double**)calloc(K + 1, sizeof(double*));
    int* hs = (int*)calloc(K + 1, sizeof(int));
    int* ws = (int*)calloc(K + 1, sizeof(int));
    hs[0] = height; ws[0] = width;
    L[0] = (double*)left; R[0] = (double*)right;
    for (int k = 1; k <= K; ++k) {
        hs[k] = (hs[k - 1] + 1) / 2; ws[k] = (ws[k - 1] + 1) / 2;
        L[k] = (double*)malloc(sizeof(double) * (size_t)hs[k] * ws[k]);
        R[k] = (double*)malloc(sizeof(double) * (size_t)hs[k] * ws[k]);
        if (hs[k - 1] < 2 || ws[k - 1] < 2) return ORC_EVALUE;
        downsample(L[k - 1], hs[k - 1], ws[k - 1], L[k]);
        downsample(R[k - 1], hs[k - 1], ws[k - 1], R[k]);
    }
    int rc = ORC_OK;
    double *dprev = NULL, *cprev = NULL;
    for (int k = K; k >= 0 && rc == ORC_OK; --k) {
        int h = hs[k], w = ws[k];
        size_t n = (size_t)h * w;
        Engine e;
        rc = engine_init(&e, L[k], R[k], h, w, level_block(block, k), level_d_max(d_max, k), sigma_eps, sign);
        if (rc) break;
        double* dk = k == 0 ? d_out : (double*)malloc(sizeof(double) * n);
        double* ck = k == 0 ? c_out : (double*)malloc(sizeof(double) * n);
        int64_t* tr = trace + (size_t)(K - k) * T_NCOLS;
        memset(tr, 0, sizeof(int64_t) * T_NCOLS);
        tr[T_LEVEL] = k;
        if (k == K) {
            rc = process_level(&e, NULL, NULL, alpha, beta, radius, dk, ck, tr);
        } else {
            double* dh = (double*)malloc(sizeof(double) * n);
            double* ch = (double*)malloc(sizeof(double) * n);
            rc = upsample_prior(dprev, cprev, hs[k + 1], ws[k + 1], h, w, dh, ch);
            if (!rc) rc = process_level(&e, dh, ch, alpha, beta, radius, dk, ck, tr);
            free(dh); free(ch);
        }
        engine_free(&e);
        if (level_d && level_c && rc == ORC_OK) {
            size_t off = 0;
            for (int t = 0; t < k; ++t) off += (size_t)hs[t] * ws[t];
            memcpy(level_d + off, dk, sizeof(double) * n);
            memcpy(level_c + off, ck, sizeof(double) * n);
        }
        free(dprev); free(cprev);
        dprev = k == 0 ? NULL : dk;
        cprev = k == 0 ? NULL : ck;
    }
    free(dprev); free(cprev);
    for (int k = 1; k <= K; ++k) { free(L[k]); free(R[k]); }
    free(L); free(R); free(hs); free(ws);
    return rc;
}

/* match_coarsest (matcher.py:184-193) for one level: first argmax over the
 * dense DSI rows.  Returns 0, or 1 for a ValueError (zncc.py:157-164). */
int mshbm_oracle_match_coarsest(const double* left, const double* right, int h, int w, int block,
                                int d_max, double sigma_eps, int sign, double* d_out,
                                double* c_out) {
    if (h < 1 || w < 1 || block < 1 || block % 2 == 0 || d_max < 0) return ORC_EVALUE;
    Engine e;
    if (engine_init(&e, left, right, h, w, block, d_max, sigma_eps, sign)) return ORC_ENOMEM;
    int rc = ORC_OK;
    #pragma omp parallel
    {
        double* row = (double*)malloc(sizeof(double) * (size_t)(d_max + 1) * w);
        double* vbuf = (double*)malloc(sizeof(double) * (size_t)(2 * (e.pw + 2 * d_max + 8)));
        if (!row || !vbuf) {
            #pragma omp atomic write
            rc = ORC_ENOMEM;
        }
        #pragma omp for schedule(dynamic, 4)
        for (int i = 0; i < h; ++i) {
            if (rc) continue;
            dsi_row(&e, i, row, vbuf);
            for (int j = 0; j < w; ++j) {
                double bc = row[j];
                int bz = 0;
                for (int z = 1; z <= d_max; ++z)
                    if (row[(size_t)z * w + j] > bc) { bc = row[(size_t)z * w + j]; bz = z; }
                d_out[(size_t)i * w + j] = (double)bz;
                c_out[(size_t)i * w + j] = bc;
            }
        }
        free(row); free(vbuf);
    }
    engine_free(&e);
    return rc;
}
