// extern "C" wrappers over the reference's OWN fscan sources — TEST
// INFRASTRUCTURE. Compiled by oracle/Makefile against /root/reference/proj
// into oracle/_ref/libfscan_ref.so; never part of the product path.
//
// Every wrapper forwards to the public reference API, unchanged:
//   scan_match            proj/src/matcher.cpp:189-216
//   magnitude/dft2        proj/src/spectral.cpp:73-117
//   hanning_window/bandpass_mask/cart2pol/rotate_bilinear
//                         proj/src/imageops.cpp:30-99
//   xcorr                 proj/src/spectral.cpp:119-153
//   soft_argmax           proj/src/matcher.cpp:57-93
//   verify suites         proj/src/verify.cpp:73,115
//   parallel_for          proj/src/parallel.cpp:24-45
//   brute_force_match     proj/src/oracle.cpp:40-67
//   write_scan/read_scan  proj/src/io.cpp:82-131 (.fscn files)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "fscan/grid.hpp"
#include "fscan/imageops.hpp"
#include "fscan/io.hpp"
#include "fscan/matcher.hpp"
#include "fscan/oracle.hpp"
#include "fscan/parallel.hpp"
#include "fscan/spectral.hpp"
#include "fscan/verify.hpp"
#include "fscan_oracle.h"

using namespace fscan;

namespace {

MatchConfig to_cfg(const fo_config* c) {
    MatchConfig m;
    m.n_theta = c->n_theta;
    m.delta_theta = c->delta_theta;
    m.t_theta = c->t_theta;
    m.n_xy = c->n_xy;
    m.delta_xy = c->delta_xy;
    m.t_xy = c->t_xy;
    m.band_lo = c->band_lo;
    m.band_hi = c->band_hi;
    m.n_radius = c->n_radius;
    m.pad_angle = c->pad_angle;
    m.softargmax_window = c->softargmax_window;
    m.normalize_scores = c->normalize_scores != 0;
    return m;
}

Array2D from_ptr(const double* p, int rows, int cols) {
    Array2D a(rows, cols);
    std::memcpy(a.data(), p, sizeof(double) * a.size());
    return a;
}

void to_ptr(const Array2D& a, double* p) { std::memcpy(p, a.data(), sizeof(double) * a.size()); }

void put_err(char* err, int len, const char* msg) {
    if (err && len > 0) std::snprintf(err, static_cast<size_t>(len), "%s", msg);
}

template <typename F>
int guard(char* err, int len, F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        put_err(err, len, e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 2;
    }
}

// Lowest linear index wins ties (the rule of matcher.cpp:46-53).
std::size_t argmax_first(const Array2D& s) {
    std::size_t best = 0;
    for (std::size_t i = 1; i < s.size(); ++i)
        if (s[i] > s[best]) best = i;
    return best;
}

void fill_result(const MatchResult& r, fo_result* out) {
    out->theta = r.pose.theta;
    out->tx = r.pose.tx;
    out->ty = r.pose.ty;
    out->theta_hard = r.diagnostics.theta_hard;
    out->theta_peak = r.diagnostics.theta_peak;
    out->xy_hard_x = r.diagnostics.xy_hard.x;
    out->xy_hard_y = r.diagnostics.xy_hard.y;
    out->xy_peak = r.diagnostics.xy_peak;
    const std::size_t tb = argmax_first(r.theta_surface.scores);
    out->theta_bin = static_cast<int>(tb / r.theta_surface.scores.cols());
    const std::size_t xb = argmax_first(r.xy_surface.scores);
    out->xy_row = static_cast<int>(xb / r.xy_surface.scores.cols());
    out->xy_col = static_cast<int>(xb % r.xy_surface.scores.cols());
    out->pad_ = 0;
}

}  // namespace

extern "C" {

int ref_band_magnitude(const double* img, int n, double band_lo, double band_hi, double* out) {
    return guard(nullptr, 0, [&] {
        const GridSpec spec{n, 1.0};
        const ScanGrid w = hanning_window(spec);
        Array2D x(n, n);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = img[i] * w.values[i];
        Array2D m = magnitude(dft2(x));
        const Array2D band = bandpass_mask(n, band_lo, band_hi);
        for (std::size_t i = 0; i < m.size(); ++i) m[i] *= band[i];
        to_ptr(m, out);
    });
}

int ref_cart2pol(const double* a, int n, int n_angle, int n_radius, double span, double* out) {
    return guard(nullptr, 0, [&] { to_ptr(cart2pol(from_ptr(a, n, n), n_angle, n_radius, span), out); });
}

int ref_rotate_bilinear(const double* g, int n, double theta, double* out) {
    return guard(nullptr, 0, [&] {
        const ScanGrid s(GridSpec{n, 1.0}, from_ptr(g, n, n));
        to_ptr(rotate_bilinear(s, theta).values, out);
    });
}

int ref_xcorr(const double* a, const double* b, int rows, int cols, double* out) {
    return guard(nullptr, 0, [&] {
        to_ptr(xcorr(from_ptr(a, rows, cols), from_ptr(b, rows, cols)).scores, out);
    });
}

int ref_soft_argmax(const double* scores, int rows, int cols, const double* row_coords,
                    const double* col_coords, double gain, int window, int normalize,
                    double* out_row, double* out_col) {
    return guard(nullptr, 0, [&] {
        CorrelationSurface s;
        s.scores = from_ptr(scores, rows, cols);
        s.row_coords.assign(row_coords, row_coords + rows);
        s.col_coords.assign(col_coords, col_coords + cols);
        const auto rc = soft_argmax(s, gain, window, normalize != 0);
        *out_row = rc.first;
        *out_col = rc.second;
    });
}

int ref_scan_match(const double* f, const double* g, const double* mf, const double* mg,
                   int n, double delta, const fo_config* cfg, fo_result* out,
                   double* theta_surface, double* xy_surface, char* err, int errlen) {
    return guard(err, errlen, [&] {
        const GridSpec spec{n, delta};
        const ScanGrid fs(spec, from_ptr(f, n, n));
        const ScanGrid gs(spec, from_ptr(g, n, n));
        const MatchConfig c = to_cfg(cfg);
        MatchResult r;
        if (mf && mg) {
            const MaskGrid mfs(spec, from_ptr(mf, n, n));
            const MaskGrid mgs(spec, from_ptr(mg, n, n));
            r = scan_match(fs, gs, c, mfs, mgs);
        } else {
            r = scan_match(fs, gs, c);
        }
        fill_result(r, out);
        if (theta_surface) to_ptr(r.theta_surface.scores, theta_surface);
        if (xy_surface) to_ptr(r.xy_surface.scores, xy_surface);
    });
}

int ref_brute_force(const double* f, const double* g, int n, double delta, const double* thetas,
                    int n_thetas, fo_bf_result* out, char* err, int errlen) {
    return guard(err, errlen, [&] {
        const GridSpec spec{n, delta};
        const ScanGrid fs(spec, from_ptr(f, n, n));
        const ScanGrid gs(spec, from_ptr(g, n, n));
        const std::vector<double> th(thetas, thetas + (n_thetas > 0 ? n_thetas : 0));
        MatchConfig cfg;  // unused by the search (oracle.cpp:48)
        const OracleResult r = brute_force_match(fs, gs, th, cfg);
        out->theta = r.pose.theta;
        out->tx = r.pose.tx;
        out->ty = r.pose.ty;
        out->score = r.score;
        // first candidate whose normalised angle is the returned one
        out->theta_index = 0;
        for (int k = 0; k < n_thetas; ++k)
            if (normalize_angle(thetas[k]) == r.pose.theta) {
                out->theta_index = k;
                break;
            }
        // cell from the back-rotated translation (exact up to rounding)
        const Vec2 d = rotate_vec(-thetas[out->theta_index], Vec2{r.pose.tx, r.pose.ty});
        const int half = (n - 1) / 2;
        out->xy_col = static_cast<int>(std::lround(d.x / delta)) + half;
        out->xy_row = static_cast<int>(std::lround(d.y / delta)) + half;
        out->pad_ = 0;
    });
}

int ref_verify(char* report, int len) {
    std::string text;
    int failures = 0;
    int rc = guard(report, len, [&] {
        for (const VerifyReport& rep : {verify_fourier_suite(), verify_oracle_suite()}) {
            for (const VerifyItem& it : rep.items) {
                text += (it.pass ? "[PASS] " : "[FAIL] ") + it.name + " " + it.detail + "\n";
                if (!it.pass) ++failures;
            }
        }
    });
    if (rc != 0) return -1;
    put_err(report, len, text.c_str());
    return failures;
}

int ref_scan_match_batch_f32(const float* f, const float* g, const float* mf, const float* mg,
                             int batch, int n, double delta, const fo_config* cfg,
                             int threads, fo_result* out) {
    std::vector<int> codes(static_cast<std::size_t>(batch), 0);
    const std::size_t nn = static_cast<std::size_t>(n) * n;
    parallel_for(0, batch, threads, [&](int k) {
        codes[k] = guard(nullptr, 0, [&] {
            const GridSpec spec{n, delta};
            Array2D fa(n, n), ga(n, n);
            for (std::size_t i = 0; i < nn; ++i) {
                fa[i] = f[k * nn + i];
                ga[i] = g[k * nn + i];
            }
            const ScanGrid fs(spec, std::move(fa));
            const ScanGrid gs(spec, std::move(ga));
            const MatchConfig c = to_cfg(cfg);
            MatchResult r;
            if (mf && mg) {
                Array2D ma(n, n), mb(n, n);
                for (std::size_t i = 0; i < nn; ++i) {
                    ma[i] = mf[k * nn + i];
                    mb[i] = mg[k * nn + i];
                }
                r = scan_match(fs, gs, c, MaskGrid(spec, std::move(ma)), MaskGrid(spec, std::move(mb)));
            } else {
                r = scan_match(fs, gs, c);
            }
            fill_result(r, &out[k]);
        });
    });
    for (int c : codes)
        if (c != 0) return c;
    return 0;
}

// .fscn writer / reader of the reference (io.cpp:82-131); values as float32
int ref_write_scan(const char* path, const float* values, int n, double delta, char* err, int errlen) {
    return guard(err, errlen, [&] {
        Array2D a(n, n);
        for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = values[i];
        write_scan(path, ScanGrid(GridSpec{n, delta}, std::move(a)));
    });
}

int ref_read_scan(const char* path, float* values, int n_max, int* n, double* delta, char* err, int errlen) {
    return guard(err, errlen, [&] {
        const ScanGrid s = read_scan(path);
        *n = s.spec.n;
        *delta = s.spec.delta;
        if (s.spec.n > n_max) throw std::runtime_error("ref_read_scan: buffer too small");
        for (std::size_t i = 0; i < s.values.size(); ++i) values[i] = static_cast<float>(s.values.data()[i]);
    });
}

}  // extern "C"
