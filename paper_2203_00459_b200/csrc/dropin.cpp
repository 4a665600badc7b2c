// dropin.cpp — the reference's C++ API (fscan/matcher.hpp, fscan/types.hpp)
// implemented on the B200 C ABI (fscan_cuda.h). Reference semantics kept:
//   scan_match / masked overload     proj/src/matcher.cpp:189-216
//   estimate_rotation / _translation matcher.cpp:95-187 (argument checks 98-101, 159-160)
//   finalize / validate              matcher.cpp:11-37 (validate without the odd-n rule, D1)
//   soft_argmax                      matcher.cpp:57-93 (host utility on a given surface)
//   geometry helpers                 proj/src/geometry.cpp:9-70
//   brute_force_match / timing_comparison   proj/src/oracle.cpp:40-101
//   trajectory helpers + odometry    proj/src/odometry.cpp:8-102, tools/main.cpp:124-135
// Single-pair calls convert the fp64 grids to fp32, run the batch pipeline on
// device 0 with a cached per-config context, and return surfaces as doubles.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <optional>
#include <cstdio>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "fscan/matcher.hpp"
#include "fscan/odometry.hpp"
#include "fscan/oracle.hpp"
#include "fscan/spectral.hpp"
#include "fscan_cuda.h"

namespace fscan {

// ---- geometry (geometry.cpp:9-70) ----

double normalize_angle(double theta) {
    theta = std::fmod(theta, 2.0 * kPi);
    if (theta <= -kPi) theta += 2.0 * kPi;
    if (theta > kPi) theta -= 2.0 * kPi;
    return theta;
}

Vec2 rotate_vec(double theta, const Vec2& x) {
    const double c = std::cos(theta), s = std::sin(theta);
    return {c * x.x - s * x.y, s * x.x + c * x.y};
}

Vec2 apply(const Pose2D& p, const Vec2& x) {
    const Vec2 r = rotate_vec(p.theta, x);
    return {r.x + p.tx, r.y + p.ty};
}

Pose2D compose(const Pose2D& a, const Pose2D& b) {
    const Vec2 t = apply(a, {b.tx, b.ty});
    return {normalize_angle(a.theta + b.theta), t.x, t.y};
}

Pose2D inverse(const Pose2D& p) {
    const Vec2 t = rotate_vec(-p.theta, {-p.tx, -p.ty});
    return {normalize_angle(-p.theta), t.x, t.y};
}

void validate(const GridSpec& spec) {
    if (spec.n <= 0) throw std::invalid_argument("GridSpec: n must be positive, got " + std::to_string(spec.n));
    if (!(spec.delta > 0.0)) throw std::invalid_argument("GridSpec: delta must be > 0");
}

std::string format_pose_csv(const Pose2D& p) {
    char buf[128];
    std::snprintf(buf, sizeof(buf), "%.17g,%.17g,%.17g", p.theta, p.tx, p.ty);
    return buf;
}

Pose2D parse_pose_csv(const std::string& line) {
    Pose2D p;
    double* out[3] = {&p.theta, &p.tx, &p.ty};
    const char* cur = line.data();
    const char* end = cur + line.size();
    for (int i = 0; i < 3; ++i) {
        while (cur != end && (*cur == ' ' || *cur == '\t')) ++cur;
        const auto r = std::from_chars(cur, end, *out[i]);
        if (r.ec != std::errc()) throw std::invalid_argument("bad pose row: '" + line + "'");
        cur = r.ptr;
        while (cur != end && (*cur == ' ' || *cur == '\t')) ++cur;
        if (i < 2) {
            if (cur == end || *cur != ',') throw std::invalid_argument("bad pose row: '" + line + "'");
            ++cur;
        }
    }
    return p;
}

// ---- config ----

namespace {

fscan_config to_c(const MatchConfig& m) {
    fscan_config c{};
    c.n_theta = m.n_theta;
    c.delta_theta = m.delta_theta;
    c.t_theta = m.t_theta;
    c.n_xy = m.n_xy;
    c.delta_xy = m.delta_xy;
    c.t_xy = m.t_xy;
    c.band_lo = m.band_lo;
    c.band_hi = m.band_hi;
    c.n_radius = m.n_radius;
    c.pad_angle = m.pad_angle;
    c.softargmax_window = m.softargmax_window;
    c.normalize_scores = m.normalize_scores ? 1 : 0;
    return c;
}

[[noreturn]] void raise(fscan_status st, const std::string& msg) {
    if (st == FSCAN_ERR_INVALID_ARGUMENT || st == FSCAN_ERR_NONFINITE || st == FSCAN_ERR_MASK_RANGE)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void check(fscan_status st, const fscan_ctx* ctx, const char* what) {
    if (st != FSCAN_OK) raise(st, std::string(what) + ": " + (ctx ? fscan_ctx_last_error(ctx) : ""));
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct CtxDeleter {
    void operator()(fscan_ctx* c) const { fscan_ctx_destroy(c); }
};

// One context per (device, config, batch capacity), cached per thread: the
// reference API is re-entrant and callers fan out over threads. The key is
// built from the named config fields (no struct padding bytes); capacities are
// rounded up to a power of two so nearby batch sizes share a context, and each
// thread keeps at most kCtxCache contexts (least recently used evicted).
constexpr std::size_t kCtxCache = 4;

std::string config_key(const fscan_config& c, int device, int cap) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%d|%a|%a|%d|%a|%a|%a|%a|%d|%d|%d|%d|dev%d|cap%d", c.n_theta, c.delta_theta,
                  c.t_theta, c.n_xy, c.delta_xy, c.t_xy, c.band_lo, c.band_hi, c.n_radius, c.pad_angle,
                  c.softargmax_window, c.normalize_scores, device, cap);
    return buf;
}

fscan_ctx* context_for(const MatchConfig& cfg, int device, int batch) {
    struct Entry {
        std::string key;
        std::unique_ptr<fscan_ctx, CtxDeleter> ctx;
    };
    thread_local std::list<Entry> cache;  // front = most recently used
    const fscan_config c = to_c(cfg);
    int cap = 1;
    while (cap < batch) cap <<= 1;
    const std::string key = config_key(c, device, cap);
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->key == key) {
            cache.splice(cache.begin(), cache, it);
            return cache.front().ctx.get();
        }
    fscan_ctx* ctx = nullptr;
    const fscan_status st = fscan_ctx_create(device, &c, cap, &ctx);
    std::unique_ptr<fscan_ctx, CtxDeleter> own(ctx);
    if (st != FSCAN_OK) raise(st, std::string("fscan_ctx_create: ") + (ctx ? fscan_ctx_last_error(ctx) : ""));
    while (cache.size() >= kCtxCache) cache.pop_back();
    cache.push_front(Entry{key, std::move(own)});
    return cache.front().ctx.get();
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { ck(cudaMalloc(&p, sizeof(T) * std::max<std::size_t>(1, n)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

std::vector<float> to_f32(const Array2D& a) {
    std::vector<float> v(a.size());
    for (std::size_t i = 0; i < a.size(); ++i) v[i] = static_cast<float>(a[i]);
    return v;
}

void upload(const Array2D& a, float* d) {
    const std::vector<float> v = to_f32(a);
    ck(cudaMemcpy(d, v.data(), sizeof(float) * v.size(), cudaMemcpyHostToDevice), "H2D");
}

CorrelationSurface theta_surface(const std::vector<double>& s, const MatchConfig& cfg) {
    CorrelationSurface out;
    out.scores = Array2D(s.size(), 1);
    for (std::size_t k = 0; k < s.size(); ++k) out.scores(k, 0) = s[k];
    out.row_coords.resize(s.size());
    if (cfg.n_theta == 1)
        out.row_coords[0] = 0.0;
    else
        for (int k = 0; k < cfg.n_theta; ++k) out.row_coords[k] = (k - cfg.n_theta / 2) * cfg.delta_theta;
    out.col_coords = {0.0};
    return out;
}

CorrelationSurface xy_surface(const std::vector<float>& s, int n, double delta) {
    CorrelationSurface out;
    out.scores = Array2D(n, n);
    for (std::size_t i = 0; i < s.size(); ++i) out.scores[i] = s[i];
    const int half = (n - 1) / 2;
    out.row_coords.resize(n);
    out.col_coords.resize(n);
    for (int i = 0; i < n; ++i) {
        out.row_coords[i] = (i - half) * delta;
        out.col_coords[i] = (i - half) * delta;
    }
    return out;
}

}  // namespace

int next_fast_size(int n) {  // spectral.cpp:155-163: strip the factors 2, 3, 5, 7
    if (n < 1) return 1;
    for (int cand = n;; ++cand) {
        int rest = cand;
        for (const int p : {2, 3, 5, 7})
            while (rest % p == 0) rest /= p;
        if (rest == 1) return cand;
    }
}

void finalize(MatchConfig& cfg) {
    fscan_config c = to_c(cfg);
    fscan_config_finalize(&c);
    cfg.n_radius = c.n_radius;
    cfg.pad_angle = c.pad_angle;
}

void validate(const MatchConfig& cfg) {
    const fscan_config c = to_c(cfg);
    char msg[256];
    if (fscan_config_validate(&c, msg, sizeof msg) != FSCAN_OK) throw std::invalid_argument(msg);
}

std::pair<double, double> soft_argmax(const CorrelationSurface& s, double gain, int window, bool normalize) {
    const int rows = (int)s.scores.rows(), cols = (int)s.scores.cols();
    if (rows == 0 || cols == 0) throw std::invalid_argument("soft_argmax: empty surface");
    if (s.row_coords.size() != (std::size_t)rows || s.col_coords.size() != (std::size_t)cols)
        throw std::invalid_argument("soft_argmax: coords do not match scores");
    std::size_t best = 0;
    for (std::size_t i = 1; i < s.scores.size(); ++i)
        if (s.scores[i] > s.scores[best]) best = i;
    const int pr = (int)(best / cols), pc = (int)(best % cols);
    const int r0 = std::max(0, pr - window), r1 = std::min(rows - 1, pr + window);
    const int c0 = std::max(0, pc - window), c1 = std::min(cols - 1, pc + window);
    double scale = 1.0;
    if (normalize) {
        double m = 0.0;
        for (int r = r0; r <= r1; ++r)
            for (int c = c0; c <= c1; ++c) m = std::max(m, std::abs(s.scores(r, c)));
        if (m > 0.0) scale = 1.0 / m;
    }
    const double top = s.scores[best] * scale;
    double ws = 0.0, rs = 0.0, cs = 0.0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            const double w = std::exp(gain * (s.scores(r, c) * scale - top));
            ws += w;
            rs += w * s.row_coords[r];
            cs += w * s.col_coords[c];
        }
    return {rs / ws, cs / ws};
}

std::pair<double, CorrelationSurface> estimate_rotation(const ScanGrid& f, const ScanGrid& g,
                                                        const MatchConfig& cfg) {
    if (!(f.spec == g.spec)) throw std::invalid_argument("estimate_rotation: grid specs differ");
    if (f.spec.n != cfg.n_xy) throw std::invalid_argument("estimate_rotation: grid size != config n_xy");
    validate(cfg);
    fscan_ctx* ctx = context_for(cfg, 0, 1);
    const int n = f.spec.n;
    DevBuf<float> df((std::size_t)n * n), dg((std::size_t)n * n);
    DevBuf<double> th(1), ts(std::max(1, cfg.n_theta));
    upload(f.values, df.p);
    upload(g.values, dg.p);
    check(fscan_estimate_rotation_batch(ctx, df.p, dg.p, 1, th.p, ts.p, nullptr), ctx, "estimate_rotation");
    double theta = 0.0;
    std::vector<double> s(std::max(1, cfg.n_theta));
    ck(cudaMemcpy(&theta, th.p, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(s.data(), ts.p, sizeof(double) * s.size(), cudaMemcpyDeviceToHost), "D2H");
    return {theta, theta_surface(s, cfg)};
}

std::pair<Vec2, CorrelationSurface> estimate_translation(const ScanGrid& f, const ScanGrid& g, double theta,
                                                         const MatchConfig& cfg) {
    if (!(f.spec == g.spec)) throw std::invalid_argument("estimate_translation: grid specs differ");
    if (f.spec.n != cfg.n_xy) {
        // the reference sizes the translation stage from the grid alone
        MatchConfig c2 = cfg;
        c2.n_xy = f.spec.n;
        c2.n_radius = c2.n_radius > 0 ? c2.n_radius : 0;
        finalize(c2);
        return estimate_translation(f, g, theta, c2);
    }
    fscan_ctx* ctx = context_for(cfg, 0, 1);
    const int n = f.spec.n;
    DevBuf<float> df((std::size_t)n * n), dg((std::size_t)n * n), xs((std::size_t)n * n);
    DevBuf<double> th(1), txy(2);
    upload(f.values, df.p);
    upload(g.values, dg.p);
    ck(cudaMemcpy(th.p, &theta, sizeof(double), cudaMemcpyHostToDevice), "H2D");
    check(fscan_estimate_translation_batch(ctx, df.p, dg.p, 1, f.spec.delta, th.p, txy.p, xs.p, nullptr), ctx,
          "estimate_translation");
    double t[2];
    std::vector<float> s((std::size_t)n * n);
    ck(cudaMemcpy(t, txy.p, sizeof t, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(s.data(), xs.p, sizeof(float) * s.size(), cudaMemcpyDeviceToHost), "D2H");
    return {Vec2{t[0], t[1]}, xy_surface(s, n, f.spec.delta)};
}

namespace {

MatchResult match_one(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg, const MaskGrid* mf,
                      const MaskGrid* mg) {
    validate(cfg);  // matcher.cpp:190
    if (!(f.spec == g.spec)) throw std::invalid_argument("scan_match: grid specs differ");
    if (mf && (!(mf->spec == f.spec) || !(mg->spec == g.spec)))
        throw std::invalid_argument("apply_mask: scan and mask specs differ");
    if (f.spec.n != cfg.n_xy) throw std::invalid_argument("estimate_rotation: grid size != config n_xy");
    fscan_ctx* ctx = context_for(cfg, 0, 1);
    const int n = f.spec.n;
    const std::size_t nn = (std::size_t)n * n;
    DevBuf<float> in(4 * nn), xs(nn);
    DevBuf<double> ts(std::max(1, cfg.n_theta));
    DevBuf<fscan_pair_result> res(1);
    upload(f.values, in.p);
    upload(g.values, in.p + nn);
    if (mf) {
        upload(mf->values, in.p + 2 * nn);
        upload(mg->values, in.p + 3 * nn);
    }
    check(fscan_match_batch(ctx, in.p, in.p + nn, mf ? in.p + 2 * nn : nullptr, mf ? in.p + 3 * nn : nullptr, 1,
                            f.spec.delta, res.p, ts.p, xs.p, nullptr),
          ctx, "scan_match");
    fscan_pair_result r;
    ck(cudaMemcpy(&r, res.p, sizeof r, cudaMemcpyDeviceToHost), "D2H");
    if (r.status != FSCAN_OK)
        raise((fscan_status)r.status, r.status == FSCAN_ERR_MASK_RANGE
                                          ? "MaskGrid: values must lie in [0, 1]"
                                          : "scan_match: input grids contain non-finite values");
    std::vector<double> s(std::max(1, cfg.n_theta));
    std::vector<float> x(nn);
    ck(cudaMemcpy(s.data(), ts.p, sizeof(double) * s.size(), cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(x.data(), xs.p, sizeof(float) * nn, cudaMemcpyDeviceToHost), "D2H");
    MatchResult out;
    out.pose = Pose2D{r.theta, r.tx, r.ty};
    out.theta_surface = theta_surface(s, cfg);
    out.xy_surface = xy_surface(x, n, f.spec.delta);
    out.diagnostics.theta_peak = r.theta_peak;
    out.diagnostics.theta_hard = r.theta_hard;
    out.diagnostics.xy_peak = r.xy_peak;
    out.diagnostics.xy_hard = Vec2{r.xy_hard_x, r.xy_hard_y};
    return out;
}

}  // namespace

MatchResult scan_match(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg) {
    return match_one(f, g, cfg, nullptr, nullptr);
}

MatchResult scan_match(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg, const MaskGrid& mask_f,
                       const MaskGrid& mask_g) {
    return match_one(f, g, cfg, &mask_f, &mask_g);
}

void scan_match_batch(const float* d_f, const float* d_g, const float* d_mf, const float* d_mg, int batch,
                      double delta, const MatchConfig& cfg, std::vector<Pose2D>& poses,
                      std::vector<PairDiagnostics>* diags, int device) {
    validate(cfg);
    poses.assign(std::max(0, batch), Pose2D{});
    if (diags) diags->assign(std::max(0, batch), PairDiagnostics{});
    if (batch <= 0) return;
    fscan_ctx* ctx = context_for(cfg, device, batch);
    DevBuf<fscan_pair_result> res(batch);
    check(fscan_match_batch(ctx, d_f, d_g, d_mf, d_mg, batch, delta, res.p, nullptr, nullptr, nullptr), ctx,
          "scan_match_batch");
    std::vector<fscan_pair_result> h(batch);
    ck(cudaMemcpy(h.data(), res.p, sizeof(fscan_pair_result) * batch, cudaMemcpyDeviceToHost), "D2H");
    for (int i = 0; i < batch; ++i) {
        if (h[i].status != FSCAN_OK)
            raise((fscan_status)h[i].status, "scan_match_batch: pair " + std::to_string(i) + " rejected");
        poses[i] = Pose2D{h[i].theta, h[i].tx, h[i].ty};
        if (diags) {
            PairDiagnostics& d = (*diags)[i];
            d.diag.theta_peak = h[i].theta_peak;
            d.diag.theta_hard = h[i].theta_hard;
            d.diag.xy_peak = h[i].xy_peak;
            d.diag.xy_hard = Vec2{h[i].xy_hard_x, h[i].xy_hard_y};
            d.theta_bin = h[i].theta_bin;
            d.xy_row = h[i].xy_row;
            d.xy_col = h[i].xy_col;
        }
    }
}

// ---- trajectories (odometry.cpp:8-102) ----

Trajectory integrate(const std::vector<Pose2D>& relatives) {
    Trajectory t;
    t.poses.reserve(relatives.size() + 1);
    t.cumulative_distance.reserve(relatives.size() + 1);
    Pose2D cur = Pose2D::identity();
    double dist = 0.0;
    t.poses.push_back(cur);
    t.cumulative_distance.push_back(dist);
    for (const Pose2D& r : relatives) {
        cur = compose(cur, r);
        dist += r.translation().norm();
        t.poses.push_back(cur);
        t.cumulative_distance.push_back(dist);
    }
    return t;
}

std::vector<Pose2D> difference(const Trajectory& t) {
    std::vector<Pose2D> out;
    for (std::size_t k = 1; k < t.poses.size(); ++k) out.push_back(compose(inverse(t.poses[k - 1]), t.poses[k]));
    return out;
}

Trajectory from_poses(std::vector<Pose2D> poses) {
    Trajectory t;
    t.poses = std::move(poses);
    double dist = 0.0;
    for (std::size_t k = 0; k < t.poses.size(); ++k) {
        if (k) dist += (t.poses[k].translation() - t.poses[k - 1].translation()).norm();
        t.cumulative_distance.push_back(dist);
    }
    return t;
}

std::optional<DriftReport> kitti_drift(const Trajectory& est, const Trajectory& truth,
                                       const std::vector<double>& lengths, int stride, DriftAveraging avg) {
    const std::size_t frames = truth.poses.size();
    if (est.poses.size() != frames) throw std::invalid_argument("kitti_drift: trajectory lengths differ");
    if (frames < 2) throw std::invalid_argument("kitti_drift: need >= 2 frames");
    if (stride < 1) throw std::invalid_argument("kitti_drift: stride must be >= 1");
    if (truth.cumulative_distance.size() != frames)
        throw std::invalid_argument("kitti_drift: truth lacks cumulative distance");
    const std::vector<double>& d = truth.cumulative_distance;
    double all_t = 0.0, all_r = 0.0, mean_t = 0.0, mean_r = 0.0;
    int all_n = 0, used_lengths = 0;
    for (const double len : lengths) {
        if (!(len > 0.0)) throw std::invalid_argument("kitti_drift: segment lengths must be positive");
        double st = 0.0, sr = 0.0;
        int cnt = 0;
        std::size_t end = 0;
        for (std::size_t first = 0; first < frames; first += stride) {
            end = std::max(end, first);  // distance is non-decreasing: the end only moves forward
            while (end < frames && d[end] - d[first] < len) ++end;
            if (end == frames) break;
            const Pose2D e = compose(inverse(compose(inverse(truth.poses[first]), truth.poses[end])),
                                     compose(inverse(est.poses[first]), est.poses[end]));
            const double seg = d[end] - d[first];
            st += e.translation().norm() / seg * 100.0;
            sr += std::abs(e.theta) * (180.0 / kPi) / (seg / 1000.0);
            ++cnt;
        }
        if (cnt) {
            all_t += st;
            all_r += sr;
            all_n += cnt;
            mean_t += st / cnt;
            mean_r += sr / cnt;
            ++used_lengths;
        }
    }
    if (!all_n) return std::nullopt;
    DriftReport r;
    r.segments = all_n;
    r.translation_percent = avg == DriftAveraging::pooled ? all_t / all_n : mean_t / used_lengths;
    r.rotation_deg_per_km = avg == DriftAveraging::pooled ? all_r / all_n : mean_r / used_lengths;
    return r;
}

std::vector<double> default_segment_lengths() { return {100, 200, 300, 400, 500, 600, 700, 800}; }

Trajectory odometry(const std::vector<ScanGrid>& scans, const MatchConfig& cfg, const std::vector<MaskGrid>* masks) {
    validate(cfg);
    if (scans.size() < 2) throw std::invalid_argument("odometry: need at least 2 scans");
    const GridSpec spec = scans[0].spec;
    for (const ScanGrid& s : scans)
        if (!(s.spec == spec)) throw std::invalid_argument("scan_match: grid specs differ");
    if (masks && masks->size() != scans.size()) throw std::invalid_argument("odometry: one mask per scan");
    if (spec.n != cfg.n_xy) throw std::invalid_argument("estimate_rotation: grid size != config n_xy");
    const int ns = (int)scans.size(), pairs = ns - 1;
    const std::size_t nn = (std::size_t)spec.n * spec.n;
    fscan_ctx* ctx = context_for(cfg, 0, pairs);
    DevBuf<float> ds(ns * nn), dm(masks ? ns * nn : 1);
    DevBuf<fscan_pair_result> res(pairs);
    for (int k = 0; k < ns; ++k) {
        upload(scans[k].values, ds.p + k * nn);
        if (masks) upload((*masks)[k].values, dm.p + k * nn);
    }
    check(fscan_odometry_batch(ctx, ds.p, masks ? dm.p : nullptr, ns, spec.delta, res.p, nullptr, nullptr, nullptr),
          ctx, "odometry");
    std::vector<fscan_pair_result> h(pairs);
    ck(cudaMemcpy(h.data(), res.p, sizeof(fscan_pair_result) * pairs, cudaMemcpyDeviceToHost), "D2H");
    std::vector<Pose2D> rels(pairs);
    for (int k = 0; k < pairs; ++k) {
        if (h[k].status != FSCAN_OK)
            raise((fscan_status)h[k].status, h[k].status == FSCAN_ERR_MASK_RANGE
                                                 ? "MaskGrid: values must lie in [0, 1]"
                                                 : "scan_match: input grids contain non-finite values");
        rels[k] = inverse(Pose2D{h[k].theta, h[k].tx, h[k].ty});  // main.cpp:131
    }
    return integrate(rels);
}

// ---- exhaustive search (oracle.cpp:40-101) ----

OracleResult brute_force_match(const ScanGrid& f, const ScanGrid& g, const std::vector<double>& thetas,
                               const MatchConfig& cfg) {
    if (!(f.spec == g.spec)) throw std::invalid_argument("brute_force_match: grid specs differ");
    if (thetas.empty()) throw std::invalid_argument("brute_force_match: empty theta candidate list");
    MatchConfig c = cfg;  // the context is sized from the grid; the search ignores the rest
    c.n_xy = f.spec.n;
    c.delta_xy = f.spec.delta;
    finalize(c);
    fscan_ctx* ctx = context_for(c, 0, 1);
    const int n = f.spec.n;
    DevBuf<float> df((std::size_t)n * n), dg((std::size_t)n * n);
    DevBuf<fscan_bf_result> res(1);
    upload(f.values, df.p);
    upload(g.values, dg.p);
    check(fscan_brute_force_batch(ctx, df.p, dg.p, 1, thetas.data(), (int)thetas.size(), f.spec.delta, res.p,
                                  nullptr),
          ctx, "brute_force_match");
    fscan_bf_result h;
    ck(cudaMemcpy(&h, res.p, sizeof h, cudaMemcpyDeviceToHost), "D2H");
    return OracleResult{Pose2D{h.theta, h.tx, h.ty}, h.score};
}

TimingComparison timing_comparison(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg, int repeats) {
    if (repeats < 10) throw std::invalid_argument("timing_comparison: repeats must be >= 10");
    std::vector<double> thetas(cfg.n_theta);
    for (int k = 0; k < cfg.n_theta; ++k) thetas[k] = (k - cfg.n_theta / 2) * cfg.delta_theta;
    auto median_of = [&](auto&& fn) {
        for (int i = 0; i < 3; ++i) fn();  // burn-in
        std::vector<double> ms(repeats);
        for (int i = 0; i < repeats; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            fn();
            ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        std::sort(ms.begin(), ms.end());
        return ms[ms.size() / 2];
    };
    TimingComparison out;
    out.repeats = repeats;
    out.matcher_median_ms = median_of([&] { (void)scan_match(f, g, cfg); });
    out.oracle_median_ms = median_of([&] { (void)brute_force_match(f, g, thetas, cfg); });
    out.ratio = out.oracle_median_ms / out.matcher_median_ms;
    return out;
}

}  // namespace fscan
