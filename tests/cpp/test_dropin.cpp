// Reference-style tests of the C++ drop-in API (include/fscan/matcher.hpp) on
// the B200. The cases follow proj/tests/test_matcher.cpp (cited per case),
// rewritten without doctest and with even grid sizes; scenes are
// Gaussian blobs rendered analytically so rotations/shifts are exact.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <limits>
#include <optional>
#include <stdexcept>
#include <vector>

#include "fscan/matcher.hpp"
#include "fscan/spectral.hpp"
#include "fscan/odometry.hpp"
#include "fscan/oracle.hpp"

using namespace fscan;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_fail;                                                                 \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);               \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                      \
    do {                                                                              \
        bool caught_ = false;                                                         \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const T&) {                                                          \
            caught_ = true;                                                           \
        } catch (...) {                                                               \
        }                                                                             \
        CHECK(caught_);                                                               \
    } while (0)

namespace {

struct Blob {
    double x, y, s, a;
};

std::vector<Blob> scene(int n, double delta, unsigned seed, int count) {
    std::vector<Blob> b;
    unsigned long long st = seed * 2654435761ull + 1;
    auto u = [&] {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        return (double)(st >> 11) * 0x1.0p-53;
    };
    const double he = 0.35 * n * delta;
    for (int i = 0; i < count; ++i) b.push_back({(2 * u() - 1) * he, (2 * u() - 1) * he, (1.5 + 1.5 * u()) * delta, 0.3 + 0.7 * u()});
    return b;
}

// Render the scene seen after pose p (objects at R(theta) q + t), GridSpec world convention.
ScanGrid render(const std::vector<Blob>& bs, const GridSpec& spec, const Pose2D& p) {
    ScanGrid g = ScanGrid::zeros(spec);
    const double c = std::cos(p.theta), s = std::sin(p.theta);
    for (int r = 0; r < spec.n; ++r)
        for (int col = 0; col < spec.n; ++col) {
            const Vec2 w = spec.cell_center(r, col);
            double v = 0.0;
            for (const Blob& b : bs) {
                const double bx = c * b.x - s * b.y + p.tx, by = s * b.x + c * b.y + p.ty;
                const double d2 = (w.x - bx) * (w.x - bx) + (w.y - by) * (w.y - by);
                v += b.a * std::exp(-d2 / (2 * b.s * b.s));
            }
            g.values(r, col) = v;
        }
    return g;
}

MatchConfig small_cfg(int n, double delta, int n_theta) {  // test_matcher.cpp:18-31
    MatchConfig cfg;
    cfg.n_xy = n;
    cfg.delta_xy = delta;
    cfg.n_theta = n_theta;
    cfg.delta_theta = kPi / n_theta;
    cfg.n_radius = 0;
    cfg.pad_angle = -1;
    cfg.band_lo = 0.15;
    finalize(cfg);
    validate(cfg);
    return cfg;
}

ScanGrid noise_scan(const GridSpec& spec, unsigned seed) {  // test_oracle.cpp:28-34
    unsigned long long st = seed * 2654435761ull + 7;
    ScanGrid out = ScanGrid::zeros(spec);
    for (std::size_t i = 0; i < out.values.size(); ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        out.values[i] = (double)(st >> 11) * 0x1.0p-53;
    }
    return out;
}

ScanGrid shift_grid(const ScanGrid& f, int dr, int dc) {  // test_oracle.cpp:36-46
    const int n = f.spec.n;
    ScanGrid out = ScanGrid::zeros(f.spec);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            const int rr = r + dr, cc = c + dc;
            if (rr >= 0 && rr < n && cc >= 0 && cc < n) out.values(rr, cc) = f.values(r, c);
        }
    return out;
}

CorrelationSurface surface_from(const Array2D& scores) {
    CorrelationSurface s;
    s.scores = scores;
    for (std::size_t r = 0; r < scores.rows(); ++r) s.row_coords.push_back(r - scores.rows() / 2.0);
    for (std::size_t c = 0; c < scores.cols(); ++c) s.col_coords.push_back(c - scores.cols() / 2.0);
    return s;
}

}  // namespace

int main() {
    // next_fast_size (test_spectral.cpp:231-240): 2^a 3^b 5^c 7^d only
    {
        CHECK(next_fast_size(1) == 1 && next_fast_size(509) == 512 && next_fast_size(511) == 512);
        CHECK(next_fast_size(1023) == 1024 && next_fast_size(2047) == 2048 && next_fast_size(11) == 12);
        CHECK(next_fast_size(13) == 14 && next_fast_size(0) == 1 && next_fast_size(97) == 98);
    }
    // config validation and derived defaults (test_matcher.cpp:60-103)
    {
        MatchConfig cfg;
        validate(cfg);
        CHECK(cfg.n_radius == 128 && cfg.pad_angle == 92);
        MatchConfig d;
        d.n_xy = 65;
        d.n_theta = 100;
        d.delta_theta = kPi / 100.0;
        d.n_radius = 0;
        d.pad_angle = -1;
        finalize(d);
        CHECK(d.n_radius == 33 && d.pad_angle == 13);
        MatchConfig bad = small_cfg(64, 0.4, 129);
        bad.band_lo = 0.8;
        CHECK_THROWS_AS(validate(bad), std::invalid_argument);
        bad = small_cfg(64, 0.4, 129);
        bad.delta_theta = kPi / 64.0;
        CHECK_THROWS_AS(validate(bad), std::invalid_argument);
        bad = small_cfg(64, 0.4, 129);
        bad.pad_angle = 129;
        CHECK_THROWS_AS(validate(bad), std::invalid_argument);
        bad = small_cfg(64, 0.4, 129);
        bad.softargmax_window = 0;
        CHECK_THROWS_AS(validate(bad), std::invalid_argument);
    }
    // soft_argmax contracts (test_matcher.cpp:105-206)
    {
        Array2D s(9, 9, 0.0);
        s(2, 6) = 5.0;
        const auto [r, c] = soft_argmax(surface_from(s), 50.0, 2, true);
        CHECK(std::abs(r - (2.0 - 4.5)) < 1e-6 && std::abs(c - (6.0 - 4.5)) < 1e-6);
        Array2D e(5, 5, 1.0);
        const auto [r2, c2] = soft_argmax(surface_from(e), 2.0, 16, true);
        CHECK(std::abs(r2 + 0.5) < 1e-9 && std::abs(c2 + 0.5) < 1e-9);
    }
    const int n = 64;
    const double delta = 0.4;
    const GridSpec spec{n, delta};
    const MatchConfig cfg = small_cfg(n, delta, 129);
    // estimate_rotation: identical grids give zero (test_matcher.cpp:210-220)
    {
        const ScanGrid f = render(scene(n, delta, 21, 14), spec, Pose2D::identity());
        const auto [theta, surface] = estimate_rotation(f, f, cfg);
        CHECK(std::abs(theta) < 1e-3);
        CHECK(surface.scores.rows() == 129 && surface.scores.cols() == 1);
        CHECK(std::abs(surface.row_coords[64]) < 1e-12);
        CHECK(std::abs(surface.row_coords[65] - surface.row_coords[64] - cfg.delta_theta) < 1e-12);
    }
    // estimate_rotation recovers a known rotation (test_matcher.cpp:222-232)
    {
        const auto bs = scene(n, delta, 33, 14);
        const ScanGrid f = render(bs, spec, Pose2D::identity());
        for (const double beta : {0.30, -0.22, 0.55}) {
            const ScanGrid g = render(bs, spec, Pose2D{beta, 0.0, 0.0});
            const auto [theta, s] = estimate_rotation(f, g, cfg);
            CHECK(std::abs(theta - beta) <= 2.0 * cfg.delta_theta);
        }
    }
    // estimate_rotation rejects mismatched inputs (test_matcher.cpp:263-271)
    {
        const ScanGrid f = ScanGrid::zeros(spec);
        const ScanGrid g = ScanGrid::zeros(GridSpec{n, 0.5});
        CHECK_THROWS_AS(estimate_rotation(f, g, cfg), std::invalid_argument);
        const ScanGrid h = ScanGrid::zeros(GridSpec{32, delta});
        CHECK_THROWS_AS(estimate_rotation(h, h, cfg), std::invalid_argument);
    }
    // estimate_translation pins an integer cell shift (test_matcher.cpp:290-300)
    {
        const auto bs = scene(n, delta, 13, 14);
        const ScanGrid f = render(bs, spec, Pose2D::identity());
        const ScanGrid g = render(bs, spec, Pose2D{0.0, 5 * delta, 3 * delta});
        const auto [t, s] = estimate_translation(f, g, 0.0, cfg);
        CHECK(std::abs(t.x - 5 * delta) < 0.25 * delta);
        CHECK(std::abs(t.y - 3 * delta) < 0.25 * delta);
        CHECK(s.scores.rows() == (std::size_t)n && s.row_coords[n / 2] > s.row_coords[n / 2 - 1]);
    }
    // scan_match recovers a rigid motion at C1 scale (test_matcher.cpp:331-347)
    {
        const int N = 256;
        const GridSpec sp{N, 0.5};
        MatchConfig c;
        c.n_xy = N;
        c.delta_xy = 0.5;
        c.n_theta = 360;
        c.delta_theta = kPi / 360;
        c.n_radius = 0;
        c.pad_angle = -1;
        finalize(c);
        const auto bs = scene(N, 0.5, 99, 60);
        const Pose2D rel{0.05, 3.2, -1.6};
        const ScanGrid f = render(bs, sp, Pose2D::identity());
        const ScanGrid g = render(bs, sp, rel);
        const MatchResult r = scan_match(f, g, c);
        CHECK(std::abs(normalize_angle(r.pose.theta - rel.theta)) <= 2.0 * c.delta_theta);
        CHECK(std::abs(r.pose.tx - rel.tx) <= sp.delta);
        CHECK(std::abs(r.pose.ty - rel.ty) <= sp.delta);
        CHECK(r.diagnostics.theta_peak >= r.theta_surface.scores(c.n_theta / 2, 0));
        CHECK(std::abs(r.diagnostics.theta_hard - rel.theta) <= 2.0 * c.delta_theta);
        // scan_match(f, g) inverts scan_match(g, f) (test_matcher.cpp:349-360)
        const Pose2D rev = inverse(scan_match(g, f, c).pose);
        CHECK(std::abs(normalize_angle(r.pose.theta - rev.theta)) <= 4.0 * c.delta_theta);
        CHECK(std::abs(r.pose.tx - rev.tx) <= sp.delta && std::abs(r.pose.ty - rev.ty) <= sp.delta);
    }
    // scan_match rejects non-finite input (test_matcher.cpp:362-372)
    {
        ScanGrid f = ScanGrid::zeros(spec), g = ScanGrid::zeros(spec);
        f.values(3, 3) = std::nan("");
        CHECK_THROWS_AS(scan_match(f, g, cfg), std::invalid_argument);
        f.values(3, 3) = 0.0;
        g.values(1, 1) = std::numeric_limits<double>::infinity();
        CHECK_THROWS_AS(scan_match(f, g, cfg), std::invalid_argument);
    }
    // masked scan_match equals matching the masked grids (test_matcher.cpp:374-387)
    {
        const auto bs = scene(n, delta, 55, 14);
        const ScanGrid f = render(bs, spec, Pose2D::identity());
        const ScanGrid g = render(bs, spec, Pose2D{0.1, 0.8, -0.4});
        Array2D mv(n, n, 1.0);
        for (int j = 0; j < n; ++j) mv(30, j) = 0.0;
        const MaskGrid m(spec, mv);
        ScanGrid fm = f, gm = g;
        for (int j = 0; j < n; ++j) fm.values(30, j) = gm.values(30, j) = 0.0;
        const Pose2D a = scan_match(f, g, cfg, m, m).pose;
        const Pose2D b = scan_match(fm, gm, cfg).pose;
        CHECK(a.theta == b.theta && a.tx == b.tx && a.ty == b.ty);
        Array2D badv(n, n, 1.0);
        badv(0, 0) = 1.5;
        CHECK_THROWS_AS(MaskGrid(spec, badv), std::invalid_argument);
    }
    // odd grid sides (the reference's own sizes, test_matcher.cpp:331-347 at n = 65)
    {
        const int n65 = 65;
        const GridSpec s65{n65, delta};
        MatchConfig c = small_cfg(n65, delta, 129);
        const auto bs = scene(n65, delta, 101, 14);
        const Pose2D rel{0.12, 0.8, -0.4};
        const ScanGrid f = render(bs, s65, Pose2D::identity());
        const ScanGrid g = render(bs, s65, rel);
        const MatchResult r = scan_match(f, g, c);
        CHECK(std::abs(normalize_angle(r.pose.theta - rel.theta)) <= 2.0 * c.delta_theta);
        CHECK(std::abs(r.pose.tx - rel.tx) <= s65.delta && std::abs(r.pose.ty - rel.ty) <= s65.delta);
        CHECK(r.xy_surface.scores.rows() == (std::size_t)n65 && r.xy_surface.scores.cols() == (std::size_t)n65);
    }
    // GPU-path limits are reported, not silently handled: sides below 33 are unsupported
    {
        MatchConfig c = small_cfg(31, delta, 65);
        const GridSpec s31{31, delta};
        const ScanGrid f = ScanGrid::zeros(s31);
        CHECK_THROWS_AS(scan_match(f, f, c), std::runtime_error);
    }
    // batched extension on device pointers
    {
        const auto bs = scene(n, delta, 7, 14);
        std::vector<float> hf(3 * n * n), hg(3 * n * n);
        const double thetas[3] = {0.0, 0.2, -0.3};
        for (int k = 0; k < 3; ++k) {
            const ScanGrid f = render(bs, spec, Pose2D::identity());
            const ScanGrid g = render(bs, spec, Pose2D{thetas[k], 0.4, -0.8});
            for (int i = 0; i < n * n; ++i) {
                hf[k * n * n + i] = (float)f.values[i];
                hg[k * n * n + i] = (float)g.values[i];
            }
        }
        float *df = nullptr, *dg = nullptr;
        cudaMalloc(&df, sizeof(float) * hf.size());
        cudaMalloc(&dg, sizeof(float) * hg.size());
        cudaMemcpy(df, hf.data(), sizeof(float) * hf.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dg, hg.data(), sizeof(float) * hg.size(), cudaMemcpyHostToDevice);
        std::vector<Pose2D> poses;
        std::vector<PairDiagnostics> diags;
        scan_match_batch(df, dg, nullptr, nullptr, 3, delta, cfg, poses, &diags);
        for (int k = 0; k < 3; ++k) {
            CHECK(std::abs(poses[k].theta - thetas[k]) <= 2.0 * cfg.delta_theta);
            CHECK(std::abs(poses[k].tx - 0.4) <= delta && std::abs(poses[k].ty + 0.8) <= delta);
        }
        cudaFree(df);
        cudaFree(dg);
    }
    // ---- exhaustive search (proj/tests/test_oracle.cpp) ----
    // self match scores the total power at the identity (test_oracle.cpp:96-110)
    {
        const GridSpec sp{64, 0.4};
        const ScanGrid f = noise_scan(sp, 4);
        const MatchConfig c = small_cfg(64, 0.4, 65);
        const OracleResult r = brute_force_match(f, f, {-0.2, 0.0, 0.2}, c);
        double sum_sq = 0.0;
        for (std::size_t i = 0; i < f.values.size(); ++i) sum_sq += f.values[i] * f.values[i];
        CHECK(r.pose.theta == 0.0 && r.pose.tx == 0.0 && r.pose.ty == 0.0);
        CHECK(std::abs(r.score - sum_sq) <= 1e-5 * sum_sq);  // fp32 path
    }
    // integer shift with a single theta candidate (test_oracle.cpp:112-122)
    {
        const GridSpec sp{64, 0.4};
        const auto bs = scene(64, 0.4, 31, 14);
        const ScanGrid f = render(bs, sp, Pose2D::identity());
        const ScanGrid g = shift_grid(f, -3, 5);  // content moved -3 rows, +5 cols
        const OracleResult r = brute_force_match(f, g, {0.0}, small_cfg(64, 0.4, 129));
        CHECK(r.pose.theta == 0.0);
        CHECK(std::abs(r.pose.tx - 5 * sp.delta) < 1e-12 && std::abs(r.pose.ty - 3 * sp.delta) < 1e-12);
    }
    // agrees with the matcher on synthetic pairs (test_oracle.cpp:136-160)
    {
        const GridSpec sp{128, 0.4};  // n = 65 there; 64 is too small for the even-n matcher
        const MatchConfig c = small_cfg(128, 0.4, 129);
        std::vector<double> ths;
        for (int k = 0; k < c.n_theta; ++k) {
            const double t = (k - c.n_theta / 2) * c.delta_theta;
            if (std::abs(t) <= 0.8) ths.push_back(t);
        }
        const Pose2D rels[3] = {{0.31, 1.2, -0.8}, {-0.22, -2.0, 0.4}, {0.05, 0.8, 2.0}};
        for (int trial = 0; trial < 3; ++trial) {
            const auto bs = scene(128, 0.4, 600 + trial, 30);
            const ScanGrid f = render(bs, sp, Pose2D::identity());
            const ScanGrid g = render(bs, sp, rels[trial]);
            const Pose2D m = scan_match(f, g, c).pose;
            const Pose2D o = brute_force_match(f, g, ths, c).pose;
            CHECK(std::abs(normalize_angle(m.theta - o.theta)) <= 2.0 * c.delta_theta);
            CHECK(std::abs(m.tx - o.tx) <= sp.delta && std::abs(m.ty - o.ty) <= sp.delta);
            std::printf("trial %d truth (%.4f %.3f %.3f) matcher (%.4f %.3f %.3f) exhaustive (%.4f %.3f %.3f)\n", trial,
                        rels[trial].theta, rels[trial].tx, rels[trial].ty, m.theta, m.tx, m.ty, o.theta, o.tx, o.ty);
        }
    }
    // input validation (test_oracle.cpp:162-167)
    {
        const GridSpec sp{64, 0.4};
        const ScanGrid f = noise_scan(sp, 1);
        const MatchConfig c = small_cfg(64, 0.4, 65);
        CHECK_THROWS_AS(brute_force_match(f, f, {}, c), std::invalid_argument);
        const ScanGrid g = noise_scan(GridSpec{64, 0.5}, 1);
        CHECK_THROWS_AS(brute_force_match(f, g, {0.0}, c), std::invalid_argument);
        CHECK_THROWS_AS(timing_comparison(f, f, c, 9), std::invalid_argument);
    }
    // timing: the exhaustive search costs more per call (test_oracle.cpp:184-196, ratio grows with n_theta)
    {
        const GridSpec sp{64, 0.4};
        const MatchConfig c = small_cfg(64, 0.4, 129);
        const auto bs = scene(64, 0.4, 77, 14);
        const ScanGrid f = render(bs, sp, Pose2D::identity());
        const ScanGrid g = render(bs, sp, Pose2D{0.1, 0.4, -0.4});
        // wall-clock medians on a shared host: up to three attempts for the ratio
        TimingComparison tc = timing_comparison(f, g, c, 10);
        for (int attempt = 1; attempt < 3 && !(tc.ratio > 1.0); ++attempt) tc = timing_comparison(f, g, c, 10);
        CHECK(tc.repeats == 10 && tc.matcher_median_ms > 0.0 && tc.oracle_median_ms > 0.0);
        CHECK(tc.ratio > 1.0);
        std::printf("timing_comparison n=64 n_theta=129: matcher %.3f ms, exhaustive %.3f ms, ratio %.1f\n",
                    tc.matcher_median_ms, tc.oracle_median_ms, tc.ratio);
    }
    // ---- trajectories (proj/tests/test_odometry.cpp) ----
    {
        auto lcg = [st = 12345ull]() mutable {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            return (double)(st >> 11) * 0x1.0p-53;
        };
        // identity relatives stand still; constant forward motion is a line (test_odometry.cpp:25-47)
        const Trajectory still = integrate(std::vector<Pose2D>(5, Pose2D::identity()));
        CHECK(still.poses.size() == 6 && still.poses.back().tx == 0.0 && still.cumulative_distance.back() == 0.0);
        const Trajectory line = integrate(std::vector<Pose2D>(10, Pose2D{0.0, 1.0, 0.0}));
        for (std::size_t k = 0; k < line.poses.size(); ++k)
            CHECK(std::abs(line.poses[k].tx - (double)k) < 1e-12 && std::abs(line.cumulative_distance[k] - (double)k) < 1e-12);
        // difference inverts integrate (49-65)
        std::vector<Pose2D> rels;
        for (int i = 0; i < 40; ++i) rels.push_back({-0.3 + 0.6 * lcg(), 0.2 + 1.8 * lcg(), -0.5 + lcg()});
        const Trajectory tr = integrate(rels);
        const std::vector<Pose2D> back = difference(tr);
        CHECK(back.size() == rels.size());
        for (std::size_t k = 0; k < rels.size(); ++k)
            CHECK(std::abs(normalize_angle(back[k].theta - rels[k].theta)) < 1e-10 &&
                  std::abs(back[k].tx - rels[k].tx) < 1e-9 && std::abs(back[k].ty - rels[k].ty) < 1e-9);
        // from_poses recomputes chord distance (67-76)
        const Trajectory ch = from_poses({Pose2D{0, 0, 0}, Pose2D{0.5, 3.0, 4.0}, Pose2D{-0.25, 3.0, 9.0}});
        CHECK(ch.cumulative_distance[1] == 5.0 && ch.cumulative_distance[2] == 10.0);
        // perfect estimate scores zero; constant bias closed form (78-107)
        const Trajectory t300 = integrate(std::vector<Pose2D>(300, Pose2D{0.0, 1.0, 0.0}));
        const auto z = kitti_drift(t300, t300, {100.0, 200.0});
        CHECK(z.has_value() && z->translation_percent == 0.0 && z->rotation_deg_per_km == 0.0 && z->segments > 0);
        const Trajectory truth = integrate(std::vector<Pose2D>(500, Pose2D{0.0, 1.0, 0.0}));
        const Trajectory est = integrate(std::vector<Pose2D>(500, Pose2D{0.0, 1.03, 0.0}));
        for (const auto avg : {DriftAveraging::pooled, DriftAveraging::per_length}) {
            const auto r = kitti_drift(est, truth, default_segment_lengths(), 1, avg);
            CHECK(r.has_value() && std::abs(r->translation_percent - 3.0) < 1e-8 && std::abs(r->rotation_deg_per_km) < 1e-9);
        }
        // invariant to a global rigid transform (109-139)
        std::vector<Pose2D> noisy = rels;
        for (Pose2D& q : noisy) {
            q.theta += 0.002 * (lcg() - 0.5);
            q.tx += 0.02 * (lcg() - 0.5);
        }
        const Trajectory et = integrate(noisy);
        const auto b0 = kitti_drift(et, tr, {5.0, 10.0});
        const Pose2D world{0.7, 100.0, -40.0};
        auto moved = [&](const Trajectory& t) {
            std::vector<Pose2D> ps;
            for (const Pose2D& q : t.poses) ps.push_back(compose(world, q));
            Trajectory o = from_poses(ps);
            o.cumulative_distance = t.cumulative_distance;
            return o;
        };
        const auto b1 = kitti_drift(moved(et), moved(tr), {5.0, 10.0});
        CHECK(b0 && b1 && std::abs(b0->translation_percent - b1->translation_percent) < 1e-9 * (1 + b0->translation_percent) &&
              b0->segments == b1->segments);
        // stride subsamples; too short is empty; validation (158-186)
        const Trajectory t200 = integrate(std::vector<Pose2D>(200, Pose2D{0.0, 1.0, 0.0}));
        const auto dense = kitti_drift(t200, t200, {50.0}, 1), sparse = kitti_drift(t200, t200, {50.0}, 10);
        CHECK(dense && sparse && dense->segments > sparse->segments && sparse->segments >= dense->segments / 10);
        const Trajectory t5 = integrate(std::vector<Pose2D>(5, Pose2D{0.0, 1.0, 0.0}));
        CHECK(!kitti_drift(t5, t5, {100.0}).has_value());
        const Trajectory a10 = integrate(std::vector<Pose2D>(10, Pose2D{0.0, 1.0, 0.0}));
        const Trajectory a11 = integrate(std::vector<Pose2D>(11, Pose2D{0.0, 1.0, 0.0}));
        CHECK_THROWS_AS(kitti_drift(a10, a11, {5.0}), std::invalid_argument);
        CHECK_THROWS_AS(kitti_drift(a10, a10, {5.0}, 0), std::invalid_argument);
        CHECK_THROWS_AS(kitti_drift(a10, a10, {-5.0}), std::invalid_argument);
        const Trajectory one = integrate({});
        CHECK_THROWS_AS(kitti_drift(one, one, {5.0}), std::invalid_argument);
        // pooled and per-length averaging differ on unevenly populated lengths (188-206)
        std::vector<Pose2D> r100(100, Pose2D{0.0, 1.0, 0.0}), e100 = r100;
        for (int i = 80; i < 100; ++i) e100[i].ty = 0.3;
        const auto po = kitti_drift(integrate(e100), integrate(r100), {10.0, 50.0}, 1, DriftAveraging::pooled);
        const auto pl = kitti_drift(integrate(e100), integrate(r100), {10.0, 50.0}, 1, DriftAveraging::per_length);
        CHECK(po && pl && std::abs(po->translation_percent - pl->translation_percent) > 1e-6);
    }
    // odometry over a rendered drive (the matching loop of main.cpp:124-135)
    {
        const int N = 128;
        const GridSpec sp{N, 0.4};
        const MatchConfig c = small_cfg(N, 0.4, 129);
        const auto bs = scene(N, 0.4, 4242, 40);
        std::vector<Pose2D> truth{Pose2D::identity()};
        const Pose2D step{0.03, 0.8, 0.2};
        for (int k = 0; k < 6; ++k) truth.push_back(compose(truth.back(), step));
        // scan k is the scene seen from pose k: objects at inverse(pose_k) applied to world points
        std::vector<ScanGrid> scans;
        for (const Pose2D& pk : truth) scans.push_back(render(bs, sp, inverse(pk)));
        const Trajectory t = odometry(scans, c);
        CHECK(t.poses.size() == truth.size());
        for (std::size_t k = 0; k < truth.size(); ++k) {
            const Pose2D e = compose(inverse(truth[k]), t.poses[k]);
            CHECK(std::abs(e.theta) <= 2.0 * (double)k * c.delta_theta + 1e-12);
            CHECK(std::abs(e.tx) <= 0.5 * k * sp.delta + 1e-12 && std::abs(e.ty) <= 0.5 * k * sp.delta + 1e-12);
        }
        // the chained batch gives the pairwise scan_match results
        for (int k = 0; k + 1 < (int)scans.size(); ++k) {
            const Pose2D m = inverse(scan_match(scans[k], scans[k + 1], c).pose);
            const Pose2D r = difference(t)[k];
            CHECK(std::abs(normalize_angle(m.theta - r.theta)) < 1e-6 && std::abs(m.tx - r.tx) < 1e-4 &&
                  std::abs(m.ty - r.ty) < 1e-4);
        }
        CHECK_THROWS_AS(odometry(std::vector<ScanGrid>(1, scans[0]), c), std::invalid_argument);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    if (g_fail == 0) std::printf("ALL PASSED\n");
    return g_fail == 0 ? 0 : 1;
}
