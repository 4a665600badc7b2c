/*
 * fscan_oracle.c — plain-C fp64 restatement of the reference hot path
 * (fscan::scan_match and the stages under it).
 *
 * TEST INFRASTRUCTURE ONLY: the checker, never the thing measured or shipped.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs load
 * oracle/liboracle.so. The product path has no CPU fallback.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference's own code compiled into oracle/_ref/ (golden vectors in
 * tests/golden/, produced by tests/golden/make_golden.py) and against the
 * reference's known-answer properties (test_spectral.cpp, test_matcher.cpp).
 * Even grid sizes follow the D1 patch: the odd-n check of
 * matcher.cpp:25 is not applied, everything else is unchanged.
 *
 * Each function mirrors the reference arithmetic in the same operation order
 * so results agree to rounding (the FFT is oracle/fft64.c in both builds).
 */
#include "fscan_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fft64.h"

typedef double complex cplx;

static const double kPi = 3.141592653589793; /* std::numbers::pi, geometry.hpp:11 */

static void set_err(char* err, int len, const char* msg) {
    if (err && len > 0) snprintf(err, (size_t)len, "%s", msg);
}

/* ---- config: matcher.cpp:11-37 ---- */

void fo_finalize(fo_config* c) {
    if (c->n_radius <= 0) c->n_radius = (c->n_xy + 1) / 2;
    if (c->pad_angle < 0) {
        const int a = (c->n_theta + 7) / 8, b = c->n_theta - 1;
        c->pad_angle = a < b ? a : b;
    }
}

int fo_validate(const fo_config* c, char* err, int len) {
    if (c->n_theta < 1) return set_err(err, len, "config: n_theta must be >= 1"), 1;
    if (!(c->delta_theta > 0.0)) return set_err(err, len, "config: delta_theta must be positive"), 1;
    if (c->n_theta * c->delta_theta > kPi + 1e-9)
        return set_err(err, len, "config: n_theta * delta_theta must not exceed pi"), 1;
    if (!(c->t_theta > 0.0) || !(c->t_xy > 0.0))
        return set_err(err, len, "config: softmax gains must be positive"), 1;
    if (c->n_xy < 3) return set_err(err, len, "config: n_xy must be >= 3"), 1; /* D1 patch */
    if (!(c->delta_xy > 0.0)) return set_err(err, len, "config: delta_xy must be positive"), 1;
    if (!(c->band_lo >= 0.0 && c->band_lo < c->band_hi && c->band_hi <= 1.0))
        return set_err(err, len, "config: band must satisfy 0 <= lo < hi <= 1"), 1;
    if (c->n_theta > 1 && c->n_radius < 2) return set_err(err, len, "config: n_radius must be >= 2"), 1;
    if (c->pad_angle < 0 || c->pad_angle >= c->n_theta)
        return set_err(err, len, "config: need 0 <= pad_angle < n_theta"), 1;
    if (c->softargmax_window < 1) return set_err(err, len, "config: softargmax_window must be >= 1"), 1;
    return 0;
}

/* spectral.cpp:155-163 */
int fo_next_fast_size(int n) {
    if (n < 1) return 1;
    for (int cand = n;; ++cand) {
        int m = cand;
        const int f[4] = {2, 3, 5, 7};
        for (int i = 0; i < 4; ++i)
            while (m % f[i] == 0) m /= f[i];
        if (m == 1) return cand;
    }
}

/* ---- imageops.cpp ---- */

/* imageops.cpp:10-26: bilinear lookup, zero fill outside the array. */
static double sample_bilinear(const double* a, long rows, long cols, double row, double col) {
    const double r0f = floor(row), c0f = floor(col);
    const long r0 = (long)r0f, c0 = (long)c0f;
    const double fr = row - r0f, fc = col - c0f;
#define AT(r, c) (((r) < 0 || (r) >= rows || (c) < 0 || (c) >= cols) ? 0.0 : a[(r) * cols + (c)])
    return (1.0 - fr) * ((1.0 - fc) * AT(r0, c0) + fc * AT(r0, c0 + 1)) +
           fr * ((1.0 - fc) * AT(r0 + 1, c0) + fc * AT(r0 + 1, c0 + 1));
#undef AT
}

/* imageops.cpp:30-42 (1-D factor; the 2-D window is w[r]*w[c]). */
static void hann_1d(int n, double* w) {
    for (int i = 0; i < n; ++i) w[i] = 1.0;
    if (n > 1)
        for (int i = 0; i < n; ++i) w[i] = 0.5 * (1.0 - cos(2.0 * kPi * i / (n - 1)));
}

/* imageops.cpp:44-59 */
static void bandpass(int n, double lo, double hi, double* out) {
    const int c = n / 2;
    const double nyq = n / 2.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double rho = hypot((double)(i - c), (double)(j - c)) / nyq;
            out[(size_t)i * n + j] = (rho >= lo && rho <= hi) ? 1.0 : 0.0;
        }
}

/* imageops.cpp:61-79 */
int fo_rotate_bilinear(const double* g, int n, double theta, double* out) {
    if (theta == 0.0) {
        memcpy(out, g, sizeof(double) * (size_t)n * n);
        return 0;
    }
    const double c = (n - 1) / 2.0;
    const double ct = cos(theta), st = sin(theta);
    for (int r = 0; r < n; ++r) {
        const double v = r - c;
        for (int col = 0; col < n; ++col) {
            const double u = col - c;
            const double src_row = c + st * u + ct * v;
            const double src_col = c + ct * u - st * v;
            out[(size_t)r * n + col] = sample_bilinear(g, n, n, src_row, src_col);
        }
    }
    return 0;
}

/* imageops.cpp:81-99 */
int fo_cart2pol(const double* a, int n, int n_angle, int n_radius, double span, double* out) {
    if (n_angle < 2 || n_radius < 2) return 1;
    const int c = n / 2;
    const double r_max = n / 2.0;
    for (int i = 0; i < n_angle; ++i) {
        const double phi = -span / 2.0 + span * i / n_angle;
        const double cp = cos(phi), sp = sin(phi);
        for (int j = 0; j < n_radius; ++j) {
            const double r = r_max * (j + 1) / n_radius;
            out[(size_t)i * n_radius + j] = sample_bilinear(a, n, n, c - r * sp, c + r * cp);
        }
    }
    return 0;
}

/* imageops.cpp:101-113 -> (na + 2p) x (nr + 2p) */
static double* wrap_pad(const double* p, int na, int nr, int pad) {
    const int rows = na + 2 * pad, cols = nr + 2 * pad;
    double* out = (double*)calloc((size_t)rows * cols, sizeof(double));
    for (int i = 0; i < rows; ++i) {
        const int src = ((i - pad) % na + na) % na;
        for (int j = 0; j < nr; ++j) out[(size_t)i * cols + j + pad] = p[(size_t)src * nr + j];
    }
    return out;
}

/* imageops.cpp:115-124 */
static double* zero_pad(const double* g, int n, int out_n) {
    const int off = (out_n - n) / 2;
    double* out = (double*)calloc((size_t)out_n * out_n, sizeof(double));
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) out[(size_t)(r + off) * out_n + c + off] = g[(size_t)r * n + c];
    return out;
}

/* ---- spectral.cpp ---- */

/* spectral.cpp:73-91 (centred forward transform) followed by
 * spectral.cpp:113-117 (modulus). */
static void dft2_magnitude(const double* g, int n, double* mag) {
    cplx* buf = (cplx*)malloc(sizeof(cplx) * (size_t)n * n);
    for (size_t i = 0; i < (size_t)n * n; ++i) buf[i] = g[i];
    fft64_exec_2d(n, n, (double*)buf, -1);
    const int h = n / 2;
    for (int r = 0; r < n; ++r) {
        const int sr = (r - h + n) % n;
        for (int c = 0; c < n; ++c)
            mag[(size_t)r * n + c] = cabs(buf[(size_t)sr * n + (c - h + n) % n]);
    }
    free(buf);
}

/* spectral.cpp:119-153: c[k] = sum_x a[x] b[x+k], zero lag at (rows/2, cols/2) */
/* phase != 0: the normalised cross-power X/|X| (0 where X = 0) before the
 * inverse — the opt-in phase correlation of SURVEY a21 (no reference code;
 * own spec). */
static int xcorr_impl(const double* a, const double* b, int rows, int cols, int phase, double* out) {
    const size_t sz = (size_t)rows * cols;
    cplx* fa = (cplx*)malloc(sizeof(cplx) * sz);
    cplx* buf = (cplx*)malloc(sizeof(cplx) * sz);
    for (size_t i = 0; i < sz; ++i) fa[i] = a[i];
    fft64_exec_2d(rows, cols, (double*)fa, -1);
    for (size_t i = 0; i < sz; ++i) buf[i] = b[i];
    fft64_exec_2d(rows, cols, (double*)buf, -1);
    for (size_t i = 0; i < sz; ++i) {
        buf[i] *= conj(fa[i]);
        if (phase) {
            const double m = cabs(buf[i]);
            buf[i] = m > 0.0 ? buf[i] / m : 0.0;
        }
    }
    fft64_exec_2d(rows, cols, (double*)buf, +1);
    const double scale = 1.0 / ((double)rows * cols);
    const int hr = rows / 2, hc = cols / 2;
    for (int r = 0; r < rows; ++r) {
        const int sr = (r - hr + rows) % rows;
        for (int c = 0; c < cols; ++c)
            out[(size_t)r * cols + c] = creal(buf[(size_t)sr * cols + (c - hc + cols) % cols]) * scale;
    }
    free(fa);
    free(buf);
    return 0;
}

int fo_xcorr(const double* a, const double* b, int rows, int cols, double* out) {
    return xcorr_impl(a, b, rows, cols, 0, out);
}

/* ---- matcher.cpp ---- */

/* matcher.cpp:47-53: strict >, lowest linear index wins. */
static size_t hard_argmax(const double* s, size_t n) {
    size_t best = 0;
    for (size_t i = 1; i < n; ++i)
        if (s[i] > s[best]) best = i;
    return best;
}

/* matcher.cpp:57-93 */
int fo_soft_argmax(const double* s, int rows, int cols, const double* rc, const double* cc,
                   double gain, int window, int normalize, double* out_row, double* out_col) {
    if (rows == 0 || cols == 0) return 1;
    const size_t best = hard_argmax(s, (size_t)rows * cols);
    const int pr = (int)(best / cols), pc = (int)(best % cols);
    const int r0 = pr - window > 0 ? pr - window : 0;
    const int r1 = pr + window < rows - 1 ? pr + window : rows - 1;
    const int c0 = pc - window > 0 ? pc - window : 0;
    const int c1 = pc + window < cols - 1 ? pc + window : cols - 1;
    double scale = 1.0;
    if (normalize) {
        double m = 0.0;
        for (int r = r0; r <= r1; ++r)
            for (int c = c0; c <= c1; ++c) {
                const double v = fabs(s[(size_t)r * cols + c]);
                m = m > v ? m : v;
            }
        if (m > 0.0) scale = 1.0 / m;
    }
    const double top = s[best] * scale;
    double wsum = 0.0, rsum = 0.0, csum = 0.0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            const double w = exp(gain * (s[(size_t)r * cols + c] * scale - top));
            wsum += w;
            rsum += w * rc[r];
            csum += w * cc[c];
        }
    *out_row = rsum / wsum;
    *out_col = csum / wsum;
    return 0;
}

/* matcher.cpp:95-153 */
int fo_estimate_rotation(const double* f, const double* g, int n, double delta,
                         const fo_config* cfg, double* theta, double* surface) {
    (void)delta;
    if (n != cfg->n_xy) return 1;
    if (cfg->n_theta == 1) {
        *theta = 0.0;
        if (surface) surface[0] = 0.0;
        return 0;
    }
    const size_t nn = (size_t)n * n;
    double* w = (double*)malloc(sizeof(double) * n);
    hann_1d(n, w);
    double* fw = (double*)malloc(sizeof(double) * nn);
    double* gw = (double*)malloc(sizeof(double) * nn);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            const double wv = w[r] * w[c];
            fw[(size_t)r * n + c] = f[(size_t)r * n + c] * wv;
            gw[(size_t)r * n + c] = g[(size_t)r * n + c] * wv;
        }
    double* band = (double*)malloc(sizeof(double) * nn);
    bandpass(n, cfg->band_lo, cfg->band_hi, band);
    double* af = (double*)malloc(sizeof(double) * nn);
    double* ag = (double*)malloc(sizeof(double) * nn);
    dft2_magnitude(fw, n, af);
    dft2_magnitude(gw, n, ag);
    for (size_t i = 0; i < nn; ++i) {
        af[i] *= band[i];
        ag[i] *= band[i];
    }
    const int nt = cfg->n_theta, nr = cfg->n_radius, pad = cfg->pad_angle;
    const double span = nt * cfg->delta_theta;
    double* pf = (double*)malloc(sizeof(double) * (size_t)nt * nr);
    double* pg = (double*)malloc(sizeof(double) * (size_t)nt * nr);
    fo_cart2pol(af, n, nt, nr, span, pf);
    fo_cart2pol(ag, n, nt, nr, span, pg);
    const int L = nt + 2 * pad, C = nr + 2 * pad;
    double *wf, *wg;
    if (pad > 0) {
        wf = wrap_pad(pf, nt, nr, pad);
        wg = wrap_pad(pg, nt, nr, pad);
    } else {
        wf = pf;
        wg = pg;
    }
    double* c2 = (double*)malloc(sizeof(double) * (size_t)L * C);
    fo_xcorr(wf, wg, L, C, c2);
    double* s = (double*)malloc(sizeof(double) * nt);
    double* rc = (double*)malloc(sizeof(double) * nt);
    for (int k = 0; k < nt; ++k) {
        double acc = 0.0;
        for (int j = 0; j < C; ++j) acc += c2[(size_t)(k + pad) * C + j];
        s[k] = acc / C;
        rc[k] = (k - nt / 2) * cfg->delta_theta;
    }
    const double cc0 = 0.0;
    double th, dummy;
    fo_soft_argmax(s, nt, 1, rc, &cc0, cfg->t_theta, cfg->softargmax_window,
                   cfg->normalize_scores, &th, &dummy);
    *theta = th;
    if (surface) memcpy(surface, s, sizeof(double) * nt);
    if (pad > 0) {
        free(wf);
        free(wg);
    }
    free(w); free(fw); free(gw); free(band); free(af); free(ag); free(pf); free(pg);
    free(c2); free(s); free(rc);
    return 0;
}

/* matcher.cpp:155-187 */
int fo_estimate_translation(const double* f, const double* g, int n, double delta,
                            double theta, const fo_config* cfg, double* tx, double* ty,
                            double* surface) {
    const size_t nn = (size_t)n * n;
    double* gr = (double*)malloc(sizeof(double) * nn);
    fo_rotate_bilinear(g, n, -theta, gr);
    const int big = fo_next_fast_size(2 * n - 1);
    double* fp = zero_pad(f, n, big);
    double* gp = zero_pad(gr, n, big);
    double* raw = (double*)malloc(sizeof(double) * (size_t)big * big);
    fo_xcorr(fp, gp, big, big, raw);
    const int h = big / 2, half = (n - 1) / 2;
    double* s = surface ? surface : (double*)malloc(sizeof(double) * nn);
    double* rc = (double*)malloc(sizeof(double) * n);
    double* cc = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        const int off_y = i - half;
        for (int j = 0; j < n; ++j) s[(size_t)i * n + j] = raw[(size_t)(h - off_y) * big + h + (j - half)];
        rc[i] = off_y * delta;
    }
    for (int j = 0; j < n; ++j) cc[j] = (j - half) * delta;
    double sy, sx;
    fo_soft_argmax(s, n, n, rc, cc, cfg->t_xy, cfg->softargmax_window, cfg->normalize_scores, &sy, &sx);
    /* rotate_vec, geometry.cpp:31-35 */
    const double c = cos(theta), sn = sin(theta);
    *tx = c * sx - sn * sy;
    *ty = sn * sx + c * sy;
    if (!surface) free(s);
    free(gr); free(fp); free(gp); free(raw); free(rc); free(cc);
    return 0;
}

/* Translation stage with a chosen padded size P (0: next_fast_size(2n-1), the
 * reference) and optional phase correlation; surface and soft-argmax as
 * estimate_translation (matcher.cpp:155-187). The GPU correlates on
 * P = 3n/2, which equals the reference's linear correlation on the kept lags
 * but not under the (size-dependent) phase normalisation: its phase-correlation
 * parity is against P = 3n/2 here. */
int fo_estimate_translation_ex(const double* f, const double* g, int n, double delta, double theta,
                               const fo_config* cfg, int pad_size, int phase, double* tx, double* ty,
                               double* surface) {
    const size_t nn = (size_t)n * n;
    double* gr = (double*)malloc(sizeof(double) * nn);
    fo_rotate_bilinear(g, n, -theta, gr);
    const int big = pad_size > 0 ? pad_size : fo_next_fast_size(2 * n - 1);
    double* fp = zero_pad(f, n, big);
    double* gp = zero_pad(gr, n, big);
    double* raw = (double*)malloc(sizeof(double) * (size_t)big * big);
    xcorr_impl(fp, gp, big, big, phase, raw);
    const int h = big / 2, half = (n - 1) / 2;
    double* s = surface ? surface : (double*)malloc(sizeof(double) * nn);
    double* rc = (double*)malloc(sizeof(double) * n);
    double* cc = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        const int off_y = i - half;
        for (int j = 0; j < n; ++j) s[(size_t)i * n + j] = raw[(size_t)(h - off_y) * big + h + (j - half)];
        rc[i] = off_y * delta;
    }
    for (int j = 0; j < n; ++j) cc[j] = (j - half) * delta;
    double sy, sx;
    fo_soft_argmax(s, n, n, rc, cc, cfg->t_xy, cfg->softargmax_window, cfg->normalize_scores, &sy, &sx);
    const double c = cos(theta), sn = sin(theta);
    *tx = c * sx - sn * sy;
    *ty = sn * sx + c * sy;
    if (!surface) free(s);
    free(gr); free(fp); free(gp); free(raw); free(rc); free(cc);
    return 0;
}

/* geometry.cpp:9-14 */
static double normalize_angle(double theta) {
    theta = fmod(theta, 2.0 * kPi);
    if (theta <= -kPi) theta += 2.0 * kPi;
    if (theta > kPi) theta -= 2.0 * kPi;
    return theta;
}

/* oracle.cpp:21-38 (score_theta) and 40-67 (brute_force_match): per candidate
 * the hard argmax of the cropped, flipped zero-padded correlation (row-major
 * scan from cell (0, 0), strict >), then the first candidate with the largest
 * score; t = rotate_vec(theta, ((col - half) delta, (row - half) delta)). */
int fo_brute_force(const double* f, const double* g, int n, double delta, const double* thetas,
                   int nth, fo_bf_result* out) {
    if (nth < 1 || n < 1) return 1;
    const size_t nn = (size_t)n * n;
    const int big = fo_next_fast_size(2 * n - 1);
    const int h = big / 2, half = (n - 1) / 2;
    double* gr = (double*)malloc(sizeof(double) * nn);
    double* raw = (double*)malloc(sizeof(double) * (size_t)big * big);
    double* fp = zero_pad(f, n, big);
    double best_score = 0.0;
    int best_k = 0, best_i = 0, best_j = 0;
    for (int k = 0; k < nth; ++k) {
        fo_rotate_bilinear(g, n, -thetas[k], gr);
        double* gp = zero_pad(gr, n, big);
        fo_xcorr(fp, gp, big, big, raw);
        free(gp);
        double b = raw[(size_t)(h + half) * big + (h - half)];
        int bi = 0, bj = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const double v = raw[(size_t)(h - (i - half)) * big + h + (j - half)];
                if (v > b) {
                    b = v;
                    bi = i;
                    bj = j;
                }
            }
        if (k == 0 || b > best_score) {
            best_score = b;
            best_k = k;
            best_i = bi;
            best_j = bj;
        }
    }
    free(gr);
    free(raw);
    free(fp);
    const double theta = thetas[best_k];
    const double dx = (best_j - half) * delta, dy = (best_i - half) * delta;
    const double c = cos(theta), sn = sin(theta);
    out->theta = normalize_angle(theta);
    out->tx = c * dx - sn * dy;
    out->ty = sn * dx + c * dy;
    out->score = best_score;
    out->theta_index = best_k;
    out->xy_row = best_i;
    out->xy_col = best_j;
    out->pad_ = 0;
    return 0;
}

int fo_band_magnitude(const double* img, int n, double lo, double hi, double* out) {
    const size_t nn = (size_t)n * n;
    double* w = (double*)malloc(sizeof(double) * n);
    hann_1d(n, w);
    double* x = (double*)malloc(sizeof(double) * nn);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) x[(size_t)r * n + c] = img[(size_t)r * n + c] * (w[r] * w[c]);
    double* band = (double*)malloc(sizeof(double) * nn);
    bandpass(n, lo, hi, band);
    dft2_magnitude(x, n, out);
    for (size_t i = 0; i < nn; ++i) out[i] *= band[i];
    free(w); free(x); free(band);
    return 0;
}

/* matcher.cpp:189-216 (+ apply_mask imageops.cpp:130-137, MaskGrid range
 * check grid.hpp:76-79, all_finite grid.hpp:83-87). */
int fo_scan_match(const double* f, const double* g, const double* mf, const double* mg,
                  int n, double delta, const fo_config* cfg, fo_result* out,
                  double* theta_surface, double* xy_surface, char* err, int errlen) {
    const size_t nn = (size_t)n * n;
    if (n <= 0 || !(delta > 0.0)) return set_err(err, errlen, "GridSpec: bad n/delta"), 1;
    double* fm = (double*)malloc(sizeof(double) * nn);
    double* gm = (double*)malloc(sizeof(double) * nn);
    int rc = 0;
    for (size_t i = 0; i < nn; ++i) {
        if (mf && mg) {
            if (!(mf[i] >= 0.0 && mf[i] <= 1.0) || !(mg[i] >= 0.0 && mg[i] <= 1.0)) {
                set_err(err, errlen, "MaskGrid: values must lie in [0, 1]");
                rc = 1;
                goto done;
            }
            fm[i] = f[i] * mf[i];
            gm[i] = g[i] * mg[i];
        } else {
            fm[i] = f[i];
            gm[i] = g[i];
        }
    }
    if ((rc = fo_validate(cfg, err, errlen)) != 0) goto done;
    for (size_t i = 0; i < nn; ++i)
        if (!isfinite(fm[i]) || !isfinite(gm[i])) {
            set_err(err, errlen, "scan_match: input grids contain non-finite values");
            rc = 1;
            goto done;
        }
    {
        const int nt = cfg->n_theta;
        double* ts = (double*)malloc(sizeof(double) * nt);
        double* xs = (double*)malloc(sizeof(double) * nn);
        double theta, tx, ty;
        if ((rc = fo_estimate_rotation(fm, gm, n, delta, cfg, &theta, ts)) != 0) {
            set_err(err, errlen, "estimate_rotation: grid size != config n_xy");
            free(ts);
            free(xs);
            goto done;
        }
        fo_estimate_translation(fm, gm, n, delta, theta, cfg, &tx, &ty, xs);
        out->theta = normalize_angle(theta);
        out->tx = tx;
        out->ty = ty;
        const size_t tb = hard_argmax(ts, (size_t)nt);
        out->theta_bin = (int)tb;
        out->theta_peak = ts[tb];
        out->theta_hard = (nt == 1) ? 0.0 : ((int)tb - nt / 2) * cfg->delta_theta;
        const size_t xb = hard_argmax(xs, nn);
        const int half = (n - 1) / 2;
        out->xy_row = (int)(xb / n);
        out->xy_col = (int)(xb % n);
        out->xy_peak = xs[xb];
        out->xy_hard_x = (out->xy_col - half) * delta;
        out->xy_hard_y = (out->xy_row - half) * delta;
        out->pad_ = 0;
        if (theta_surface) memcpy(theta_surface, ts, sizeof(double) * nt);
        if (xy_surface) memcpy(xy_surface, xs, sizeof(double) * nn);
        free(ts);
        free(xs);
    }
done:
    free(fm);
    free(gm);
    return rc;
}

/* Polar sweep -> Cartesian grid (no reference exists, parity
 * unpinned). Spec: cell (r, c) sits at world
 * x = (c - (n-1)/2) * delta, y = -(r - (n-1)/2) * delta (integer (n-1)/2, the
 * GridSpec convention of geometry.hpp:55); azimuth bin a is centred on
 * phi = 2*pi*a/n_az (CCW from +x, wrapping), range bin k on (k + 0.5) * res.
 * Bilinear in (azimuth, range); range taps outside [0, n_range) are zero. */
int fo_polar_to_cart(const double* polar, int n_az, int n_range, double res, int n,
                     double delta, double* out) {
    const int half = (n - 1) / 2;
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            const double x = (c - half) * delta;
            const double y = -((r - half) * delta);
            const double rho = sqrt(x * x + y * y);
            double phi = atan2(y, x);
            if (phi < 0.0) phi += 2.0 * kPi;
            double fa = phi * (n_az / (2.0 * kPi));
            const double fk = rho / res - 0.5;
            double a0f = floor(fa);
            const double wa = fa - a0f;
            long a0 = (long)a0f % n_az;
            const long a1 = (a0 + 1) % n_az;
            const double k0f = floor(fk);
            const long k0 = (long)k0f;
            const double wk = fk - k0f;
#define PT(a, k) (((k) < 0 || (k) >= n_range) ? 0.0 : polar[(size_t)(a) * n_range + (k)])
            out[(size_t)r * n + c] = (1.0 - wa) * ((1.0 - wk) * PT(a0, k0) + wk * PT(a0, k0 + 1)) +
                                     wa * ((1.0 - wk) * PT(a1, k0) + wk * PT(a1, k0 + 1));
#undef PT
        }
    return 0;
}
