// Host side of the synthetic scan-pair generator (include/fscan_synth.h): scene
// construction, CPU renderers and the fscan_synth_* host entry points. Pure C++
// (no CUDA): the same source is compiled into the product library and, by
// oracle/Makefile, into the CPU reference arm's input generator, so both arms
// of bench.py register byte-identical host-rendered inputs.
//
// builds inputs for tests and the bench outside any timed region.
//
// Scene model (BASELINE.json configs; SURVEY.md §8(d) "[assume]" items are
// documented in DESIGN.md §4):
//   * n_reflectors Gaussian point reflectors, centre uniform over the central
//     extent_frac of the grid, sigma ~ U(sigma_lo, sigma_hi) cells, amp ~ U(.5, 1)
//   * n_segments Gaussian line segments (endpoints in the same box,
//     cross-section sigma seg_sigma cells, amp ~ U(.5, 1))
//   * scan B renders the same objects moved by the pose p (apply(p, q)),
//     evaluated analytically (no resampling), with fresh speckle
//   * additive Rayleigh speckle; polar sweeps attenuate returns with range
//   * masks: box5x5(sigmoid(N(0, mask_sigma))), clamp-to-edge border
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "fscan_synth.h"
#include "synth_common.h"
#include "synth_scene.h"

using fsynth::Object;
using fsynth::PairScene;

namespace fsynth {

void build_scene(const fscan_synth_spec& s, int pair, PairScene* out) {
    fsynth::Seq rng(fsynth::stream_key(s.seed, (uint64_t)pair, 0, 7));
    out->theta = rng.uniform(-s.theta_max, s.theta_max);
    out->tx = rng.uniform(-s.t_max, s.t_max);
    out->ty = rng.uniform(-s.t_max, s.t_max);
    const double he = 0.5 * s.extent_frac * s.n * s.delta;
    out->a.clear();
    out->b.clear();
    auto add = [&](double x0, double y0, double x1, double y1, double sigma, double amp) {
        Object o;
        o.x0 = x0;
        o.y0 = y0;
        o.x1 = x1;
        o.y1 = y1;
        o.inv2s2 = 1.0 / (2.0 * sigma * sigma);
        o.cut2 = 25.0 * sigma * sigma;
        o.amp = amp;
        out->a.push_back(o);
    };
    for (int i = 0; i < s.n_reflectors; ++i) {
        const double cx = rng.uniform(-he, he), cy = rng.uniform(-he, he);
        const double sg = rng.uniform(s.sigma_lo_px, s.sigma_hi_px) * s.delta;
        const double amp = rng.uniform(0.5, 1.0);
        add(cx, cy, cx, cy, sg, amp);
    }
    for (int i = 0; i < s.n_segments; ++i) {
        const double x0 = rng.uniform(-he, he), y0 = rng.uniform(-he, he);
        const double x1 = rng.uniform(-he, he), y1 = rng.uniform(-he, he);
        const double amp = rng.uniform(0.5, 1.0);
        add(x0, y0, x1, y1, s.seg_sigma_px * s.delta, amp);
    }
    const double c = std::cos(out->theta), sn = std::sin(out->theta);
    for (Object o : out->a) {  // B = objects moved by p: R(theta) q + t
        const double x0 = c * o.x0 - sn * o.y0 + out->tx, y0 = sn * o.x0 + c * o.y0 + out->ty;
        const double x1 = c * o.x1 - sn * o.y1 + out->tx, y1 = sn * o.x1 + c * o.y1 + out->ty;
        o.x0 = x0;
        o.y0 = y0;
        o.x1 = x1;
        o.y1 = y1;
        out->b.push_back(o);
    }
}

// the scene of pair `seq`, with its objects moved by pose P_k, P_0 = identity
// and P_k (k > 0) the pose pair seq + k would use: independent bounded poses,
// so consecutive scans differ by at most twice the pair pose range.
void sequence_scan(const fscan_synth_spec& s, int seq, int k, const PairScene& base, std::vector<Object>* out,
                   double* pose) {
    double th = 0.0, tx = 0.0, ty = 0.0;
    if (k > 0) {
        PairScene pk;
        build_scene(s, seq + k, &pk);
        th = pk.theta;
        tx = pk.tx;
        ty = pk.ty;
    }
    const double c = std::cos(th), sn = std::sin(th);
    out->clear();
    for (Object o : base.a) {
        const double x0 = c * o.x0 - sn * o.y0 + tx, y0 = sn * o.x0 + c * o.y0 + ty;
        const double x1 = c * o.x1 - sn * o.y1 + tx, y1 = sn * o.x1 + c * o.y1 + ty;
        o.x0 = x0;
        o.y0 = y0;
        o.x1 = x1;
        o.y1 = y1;
        out->push_back(o);
    }
    if (pose) {
        pose[0] = th;
        pose[1] = tx;
        pose[2] = ty;
    }
}

}  // namespace fsynth

namespace {

using fsynth::build_scene;

struct Bbox {
    double xlo, xhi, ylo, yhi;
};

Bbox bbox(const Object& o) {
    const double cut = std::sqrt(o.cut2);
    return {std::min(o.x0, o.x1) - cut, std::max(o.x0, o.x1) + cut, std::min(o.y0, o.y1) - cut,
            std::max(o.y0, o.y1) + cut};
}

// Cartesian render of one scan (objects splatted in order, then speckle).
void render_cart_host(const fscan_synth_spec& s, const std::vector<Object>& objs, int pair, int scan,
                      float* out) {
    const int n = s.n;
    std::vector<double> acc((size_t)n * n, 0.0);
    const int half = (n - 1) / 2;
    for (const Object& o : objs) {
        const Bbox b = bbox(o);
        // x = (c - half) delta, y = -(r - half) delta
        const int c0 = std::max(0, (int)std::floor(b.xlo / s.delta) + half - 1);
        const int c1 = std::min(n - 1, (int)std::ceil(b.xhi / s.delta) + half + 1);
        const int r0 = std::max(0, half - (int)std::ceil(b.yhi / s.delta) - 1);
        const int r1 = std::min(n - 1, half - (int)std::floor(b.ylo / s.delta) + 1);
        for (int r = r0; r <= r1; ++r)
            for (int cc = c0; cc <= c1; ++cc) {
                double x, y;
                fsynth::cell_world(n, s.delta, r, cc, &x, &y);
                acc[(size_t)r * n + cc] += fsynth::object_value(o, x, y);
            }
    }
    const uint64_t key = fsynth::stream_key(s.seed, (uint64_t)pair, (uint64_t)scan, 1);
    for (size_t i = 0; i < acc.size(); ++i)
        out[i] = (float)(acc[i] + fsynth::rayleigh(key, i, s.speckle));
}

void render_polar_host(const fscan_synth_spec& s, const std::vector<Object>& objs, int pair,
                       int scan, float* out) {
    std::vector<Bbox> boxes;
    for (const Object& o : objs) boxes.push_back(bbox(o));
    const uint64_t key = fsynth::stream_key(s.seed, (uint64_t)pair, (uint64_t)scan, 1);
    for (int a = 0; a < s.n_az; ++a) {
        const double phi = 2.0 * fsynth::kPi * a / s.n_az;
        const double cp = std::cos(phi), sp = std::sin(phi);
        for (int k = 0; k < s.n_range; ++k) {
            const double rho = (k + 0.5) * s.range_res;
            const double x = rho * cp, y = rho * sp;
            double v = 0.0;
            for (size_t i = 0; i < objs.size(); ++i) {
                const Bbox& b = boxes[i];
                if (x < b.xlo || x > b.xhi || y < b.ylo || y > b.yhi) continue;
                v += fsynth::object_value(objs[i], x, y);
            }
            const double att = s.att_r0 / std::max(rho, s.att_r0);
            const size_t idx = (size_t)a * s.n_range + k;
            out[idx] = (float)(v * att * att + fsynth::rayleigh(key, idx, s.speckle));
        }
    }
}

void mask_host(const fscan_synth_spec& s, int pair, int scan, float* out) {
    const int n = s.n;
    std::vector<double> sg((size_t)n * n);
    const uint64_t key = fsynth::stream_key(s.seed, (uint64_t)pair, (uint64_t)scan, 2);
    for (size_t i = 0; i < sg.size(); ++i) sg[i] = fsynth::sigmoid(s.mask_sigma * fsynth::normal(key, i));
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            double acc = 0.0;
            for (int dr = -2; dr <= 2; ++dr)
                for (int dc = -2; dc <= 2; ++dc) {
                    const int rr = std::min(n - 1, std::max(0, r + dr));
                    const int cc = std::min(n - 1, std::max(0, c + dc));
                    acc += sg[(size_t)rr * n + cc];
                }
            out[(size_t)r * n + c] = (float)(acc / 25.0);
        }
}

template <typename F>
void parallel_pairs(int count, int threads, F&& fn) {
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = std::max(1, std::min(threads, count));
    if (threads == 1) {
        for (int i = 0; i < count; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (int i = t; i < count; i += threads) fn(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int fscan_synth_preset(int id, fscan_synth_spec* o) {
    std::memset(o, 0, sizeof(*o));
    const double deg = fsynth::kPi / 180.0;
    o->n_reflectors = 40;
    o->n_segments = 10;
    o->sigma_lo_px = 1.0;
    o->sigma_hi_px = 3.0;
    o->seg_sigma_px = 1.0;
    o->extent_frac = 0.7;
    o->theta_max = 5.0 * deg;
    o->speckle = 0.1;
    o->mask_sigma = 2.0;
    o->att_r0 = 10.0;
    o->seed = 220300459ull;
    switch (id) {
        case 1:
        case 2:
            o->n = 256;
            o->delta = 0.5;
            o->t_max = 8 * 0.5;
            o->masks = (id == 2);
            return 0;
        case 3:
        case 4:
            o->polar = 1;
            o->n = 512;
            o->delta = 0.25;
            o->t_max = 4.0;
            o->masks = 1;
            o->n_az = 400;
            o->n_range = 3768;
            o->range_res = 0.0438;
            return 0;
        case 5:
            o->n = 1024;
            o->delta = 0.125;
            o->n_reflectors = 640;
            o->n_segments = 160;
            o->theta_max = 10.0 * deg;
            o->t_max = 32 * 0.125;
            o->masks = 1;
            return 0;
        default:
            return -1;
    }
}

int fscan_synth_polar_host(const fscan_synth_spec* s, int first, int count, float* pf, float* pg,
                           double* truth, int threads) {
    if (!s->polar) return -1;
    const size_t np = (size_t)s->n_az * s->n_range;
    parallel_pairs(count, threads, [&](int i) {
        PairScene ps;
        build_scene(*s, first + i, &ps);
        render_polar_host(*s, ps.a, first + i, 0, pf + i * np);
        render_polar_host(*s, ps.b, first + i, 1, pg + i * np);
        if (truth) {
            truth[3 * i] = ps.theta;
            truth[3 * i + 1] = ps.tx;
            truth[3 * i + 2] = ps.ty;
        }
    });
    return 0;
}

int fscan_synth_pairs_host(const fscan_synth_spec* s, int first, int count, float* f, float* g,
                           float* mf, float* mg, double* truth, int threads) {
    const size_t nn = (size_t)s->n * s->n;
    parallel_pairs(count, threads, [&](int i) {
        PairScene ps;
        build_scene(*s, first + i, &ps);
        if (s->polar) {
            const size_t np = (size_t)s->n_az * s->n_range;
            std::vector<float> pa(np), pb(np);
            render_polar_host(*s, ps.a, first + i, 0, pa.data());
            render_polar_host(*s, ps.b, first + i, 1, pb.data());
            for (int r = 0; r < s->n; ++r)
                for (int c = 0; c < s->n; ++c) {
                    f[i * nn + (size_t)r * s->n + c] = (float)fscan_k0::polar_cell(
                        pa.data(), s->n_az, s->n_range, s->range_res, s->n, s->delta, r, c);
                    g[i * nn + (size_t)r * s->n + c] = (float)fscan_k0::polar_cell(
                        pb.data(), s->n_az, s->n_range, s->range_res, s->n, s->delta, r, c);
                }
        } else {
            render_cart_host(*s, ps.a, first + i, 0, f + i * nn);
            render_cart_host(*s, ps.b, first + i, 1, g + i * nn);
        }
        if (mf && mg) {
            if (s->masks) {
                mask_host(*s, first + i, 0, mf + i * nn);
                mask_host(*s, first + i, 1, mg + i * nn);
            } else {
                std::fill(mf + i * nn, mf + (i + 1) * nn, 1.0f);
                std::fill(mg + i * nn, mg + (i + 1) * nn, 1.0f);
            }
        }
        if (truth) {
            truth[3 * i] = ps.theta;
            truth[3 * i + 1] = ps.tx;
            truth[3 * i + 2] = ps.ty;
        }
    });
    return 0;
}

}  // extern "C"
