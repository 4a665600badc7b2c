// Synthetic scan-pair generator (include/fscan_synth.h). Harness code: it
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
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "fscan_synth.h"
#include "synth_common.h"

namespace fscan_detail {
// Product K0 kernel launcher (kernels.cu); used to turn device-rendered polar
// sweeps into Cartesian scans the same way the C3 hot path does.
cudaError_t launch_polar_to_cart(const float* d_polar0, const float* d_polar1, int batch, int n_az,
                                 int n_range, double range_res, int n, double delta, float* d_out0,
                                 float* d_out1, cudaStream_t stream, const void* tab);
}  // namespace fscan_detail

using fsynth::Object;

namespace {

struct PairScene {
    std::vector<Object> a, b;
    double theta = 0, tx = 0, ty = 0;
};

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

// ---- device renderers ----

constexpr int kTile = 16;

// One CTA per 16x16 tile of one scan; objects staged through shared memory in
// order so each cell sums them in the host renderer's order.
__global__ void render_cart_kernel(const Object* objs, const int* obj_off, int n, double delta,
                                   uint64_t seed, double speckle, int first, float* out_a,
                                   float* out_b) {
    __shared__ Object sh[128];
    const int scan_idx = blockIdx.z;  // 2 * local pair + scan
    const int lp = scan_idx >> 1, scan = scan_idx & 1;
    const int r = blockIdx.y * kTile + threadIdx.y;
    const int c = blockIdx.x * kTile + threadIdx.x;
    const int o0 = obj_off[scan_idx], o1 = obj_off[scan_idx + 1];
    double x, y;
    fsynth::cell_world(n, delta, r, c, &x, &y);
    double acc = 0.0;
    const int tid = threadIdx.y * kTile + threadIdx.x;
    for (int base = o0; base < o1; base += 128) {
        const int cnt = min(128, o1 - base);
        __syncthreads();
        if (tid < cnt) sh[tid] = objs[base + tid];
        __syncthreads();
        if (r < n && c < n)
            for (int i = 0; i < cnt; ++i) acc += fsynth::object_value(sh[i], x, y);
    }
    if (r < n && c < n) {
        const uint64_t key = fsynth::stream_key(seed, (uint64_t)(first + lp), (uint64_t)scan, 1);
        const size_t idx = (size_t)r * n + c;
        float* out = scan ? out_b : out_a;
        out[(size_t)lp * n * n + idx] = (float)(acc + fsynth::rayleigh(key, idx, speckle));
    }
}

__global__ void render_polar_kernel(const Object* objs, const int* obj_off, int n_az, int n_range,
                                    double res, double att_r0, uint64_t seed, double speckle,
                                    int first, float* out_a, float* out_b) {
    __shared__ Object sh[128];
    const int scan_idx = blockIdx.z;
    const int lp = scan_idx >> 1, scan = scan_idx & 1;
    const int a = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int o0 = obj_off[scan_idx], o1 = obj_off[scan_idx + 1];
    const double phi = 2.0 * fsynth::kPi * a / n_az;
    const double rho = (k + 0.5) * res;
    double sp, cp;
    sincos(phi, &sp, &cp);
    const double x = rho * cp, y = rho * sp;
    double v = 0.0;
    for (int base = o0; base < o1; base += 128) {
        const int cnt = min(128, o1 - base);
        __syncthreads();
        if ((int)threadIdx.x < cnt) sh[threadIdx.x] = objs[base + threadIdx.x];
        __syncthreads();
        if (k < n_range)
            for (int i = 0; i < cnt; ++i) v += fsynth::object_value(sh[i], x, y);
    }
    if (k < n_range) {
        const double att = att_r0 / fmax(rho, att_r0);
        const uint64_t key = fsynth::stream_key(seed, (uint64_t)(first + lp), (uint64_t)scan, 1);
        const size_t idx = (size_t)a * n_range + k;
        float* out = scan ? out_b : out_a;
        out[(size_t)lp * n_az * n_range + idx] = (float)(v * att * att + fsynth::rayleigh(key, idx, speckle));
    }
}

__global__ void mask_sigmoid_kernel(int n, uint64_t seed, double sigma, int first, float* tmp) {
    const int scan_idx = blockIdx.y;
    const int lp = scan_idx >> 1, scan = scan_idx & 1;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n * n) return;
    const uint64_t key = fsynth::stream_key(seed, (uint64_t)(first + lp), (uint64_t)scan, 2);
    tmp[(size_t)scan_idx * n * n + i] = (float)fsynth::sigmoid(sigma * fsynth::normal(key, i));
}

// box 5x5 with clamp-to-edge; tmp holds fp32 sigmoid values (the host keeps
// them in double, a <= 1 ulp difference in the mask).
__global__ void mask_box_kernel(int n, const float* tmp, float* mf, float* mg) {
    const int scan_idx = blockIdx.y;
    const int lp = scan_idx >> 1, scan = scan_idx & 1;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n * n) return;
    const int r = (int)(i / n), c = (int)(i % n);
    const float* src = tmp + (size_t)scan_idx * n * n;
    double acc = 0.0;
    for (int dr = -2; dr <= 2; ++dr)
        for (int dc = -2; dc <= 2; ++dc) {
            const int rr = min(n - 1, max(0, r + dr));
            const int cc = min(n - 1, max(0, c + dc));
            acc += src[(size_t)rr * n + cc];
        }
    float* out = scan ? mg : mf;
    out[(size_t)lp * n * n + i] = (float)(acc / 25.0);
}

__global__ void fill_ones_kernel(float* p, size_t count) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = 1.0f;
}

// Sequence mode (seq >= 0): scan k (= 2 * local pair + scan) of ONE scene,
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

// Upload per-scan object lists (scan_idx = 2 * local pair + scan).
cudaError_t upload_scenes(const fscan_synth_spec& s, int first, int count, double* truth,
                          cudaStream_t st, Object** d_objs, int** d_off, int seq = -1) {
    std::vector<Object> all;
    std::vector<int> off(1, 0);
    PairScene ps, base;
    std::vector<Object> tmp;
    if (seq >= 0) build_scene(s, seq, &base);
    for (int i = 0; i < count; ++i) {
        if (seq >= 0) {  // truth: the absolute pose of every scan
            for (int sc = 0; sc < 2; ++sc) {
                sequence_scan(s, seq, 2 * (first + i) + sc, base, &tmp, truth ? truth + 6 * i + 3 * sc : nullptr);
                all.insert(all.end(), tmp.begin(), tmp.end());
                off.push_back((int)all.size());
            }
            continue;
        }
        build_scene(s, first + i, &ps);
        all.insert(all.end(), ps.a.begin(), ps.a.end());
        off.push_back((int)all.size());
        all.insert(all.end(), ps.b.begin(), ps.b.end());
        off.push_back((int)all.size());
        if (truth) {
            truth[3 * i] = ps.theta;
            truth[3 * i + 1] = ps.tx;
            truth[3 * i + 2] = ps.ty;
        }
    }
    cudaError_t e = cudaMalloc(d_objs, sizeof(Object) * std::max<size_t>(1, all.size()));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(d_off, sizeof(int) * off.size());
    if (e != cudaSuccess) return e;
    if (!all.empty())
        e = cudaMemcpyAsync(*d_objs, all.data(), sizeof(Object) * all.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(*d_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);  // host vectors go out of scope
}

cudaError_t device_masks(const fscan_synth_spec& s, int first, int count, float* mf, float* mg,
                         cudaStream_t st) {
    const size_t nn = (size_t)s.n * s.n;
    const int threads = 256;
    if (!s.masks) {
        const size_t total = nn * count;
        fill_ones_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, st>>>(mf, total);
        fill_ones_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, st>>>(mg, total);
        return cudaGetLastError();
    }
    // chunk so the fp32 temp stays bounded
    const int chunk = std::max(1, std::min(count, (int)((256ull << 20) / (2 * nn * sizeof(float)))));
    float* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, 2 * nn * sizeof(float) * chunk);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < count; i += chunk) {
        const int cnt = std::min(chunk, count - i);
        dim3 grid((unsigned)((nn + threads - 1) / threads), 2 * cnt);
        mask_sigmoid_kernel<<<grid, threads, 0, st>>>(s.n, s.seed, s.mask_sigma, first + i, tmp);
        mask_box_kernel<<<grid, threads, 0, st>>>(s.n, tmp, mf + i * nn, mg + i * nn);
    }
    e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    return e == cudaSuccess ? cudaGetLastError() : e;
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

static int polar_device(const fscan_synth_spec* s, int first, int count, float* d_pf, float* d_pg,
                        double* truth, void* stream, int seq) {
    if (!s->polar) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    Object* objs = nullptr;
    int* off = nullptr;
    cudaError_t e = upload_scenes(*s, first, count, truth, st, &objs, &off, seq);
    if (e == cudaSuccess) {
        // gridDim.z <= 65535 scans per launch
        const int per = 16384;
        for (int i = 0; i < count && e == cudaSuccess; i += per) {
            const int cnt = std::min(per, count - i);
            dim3 grid((unsigned)((s->n_range + 127) / 128), (unsigned)s->n_az, (unsigned)(2 * cnt));
            const size_t np = (size_t)s->n_az * s->n_range;
            render_polar_kernel<<<grid, 128, 0, st>>>(objs, off + 2 * i, s->n_az, s->n_range, s->range_res,
                                                      s->att_r0, s->seed, s->speckle, first + i,
                                                      d_pf + i * np, d_pg + i * np);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFree(objs);
    cudaFree(off);
    return e == cudaSuccess ? 0 : (int)e;
}

int fscan_synth_polar_device(const fscan_synth_spec* s, int first, int count, float* d_pf,
                             float* d_pg, double* truth, void* stream) {
    return polar_device(s, first, count, d_pf, d_pg, truth, stream, -1);
}

static int pairs_device(const fscan_synth_spec* s, int first, int count, float* d_f, float* d_g, float* d_mf,
                        float* d_mg, double* truth, void* stream, int seq) {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nn = (size_t)s->n * s->n;
    cudaError_t e = cudaSuccess;
    if (s->polar) {
        const size_t np = (size_t)s->n_az * s->n_range;
        const int chunk = std::max(1, std::min(count, 64));
        float *pa = nullptr, *pb = nullptr;
        e = cudaMalloc(&pa, np * sizeof(float) * chunk);
        if (e == cudaSuccess) e = cudaMalloc(&pb, np * sizeof(float) * chunk);
        for (int i = 0; i < count && e == cudaSuccess; i += chunk) {
            const int cnt = std::min(chunk, count - i);
            const int rc = polar_device(s, first + i, cnt, pa, pb,
                                        truth ? truth + (seq >= 0 ? 6 : 3) * i : nullptr, st, seq);
            if (rc != 0) {
                e = (cudaError_t)rc;
                break;
            }
            e = fscan_detail::launch_polar_to_cart(pa, pb, cnt, s->n_az, s->n_range, s->range_res, s->n, s->delta,
                                                   d_f + i * nn, d_g + i * nn, st, nullptr);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
        cudaFree(pa);
        cudaFree(pb);
    } else {
        Object* objs = nullptr;
        int* off = nullptr;
        e = upload_scenes(*s, first, count, truth, st, &objs, &off, seq);
        const int per = 16384;
        for (int i = 0; i < count && e == cudaSuccess; i += per) {
            const int cnt = std::min(per, count - i);
            dim3 grid((unsigned)((s->n + kTile - 1) / kTile), (unsigned)((s->n + kTile - 1) / kTile),
                      (unsigned)(2 * cnt));
            render_cart_kernel<<<grid, dim3(kTile, kTile), 0, st>>>(objs, off + 2 * i, s->n, s->delta, s->seed,
                                                                    s->speckle, first + i, d_f + i * nn,
                                                                    d_g + i * nn);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        cudaFree(objs);
        cudaFree(off);
    }
    if (e == cudaSuccess && d_mf && d_mg) e = device_masks(*s, first, count, d_mf, d_mg, st);
    return e == cudaSuccess ? 0 : (int)e;
}

int fscan_synth_pairs_device(const fscan_synth_spec* s, int first, int count, float* d_f, float* d_g,
                             float* d_mf, float* d_mg, double* truth, void* stream) {
    return pairs_device(s, first, count, d_f, d_g, d_mf, d_mg, truth, stream, -1);
}

int fscan_synth_sequence_device(const fscan_synth_spec* s, int seq, int count, float* d_scans, float* d_masks,
                                double* truth, void* stream) {
    if (count < 1 || seq < 0) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nn = (size_t)s->n * s->n;
    const int pairs = (count + 1) / 2;  // rendered as pairs (even scans, odd scans), then interleaved
    float *ev = nullptr, *od = nullptr, *mev = nullptr, *mod = nullptr;
    std::vector<double> tr(truth ? 6 * (size_t)pairs : 0);
    cudaError_t e = cudaMalloc(&ev, 2 * nn * sizeof(float) * pairs);
    if (e == cudaSuccess && d_masks) e = cudaMalloc(&mev, 2 * nn * sizeof(float) * pairs);
    od = ev + nn * pairs;
    if (mev) mod = mev + nn * pairs;
    int rc = e == cudaSuccess ? pairs_device(s, 0, pairs, ev, od, mev, mod, truth ? tr.data() : nullptr, st, seq)
                              : (int)e;
    if (rc == 0) {
        const size_t row = nn * sizeof(float);
        e = cudaMemcpy2DAsync(d_scans, 2 * row, ev, row, row, pairs, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && count / 2)
            e = cudaMemcpy2DAsync(d_scans + nn, 2 * row, od, row, row, count / 2, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && d_masks)
            e = cudaMemcpy2DAsync(d_masks, 2 * row, mev, row, row, pairs, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && d_masks && count / 2)
            e = cudaMemcpy2DAsync(d_masks + nn, 2 * row, mod, row, row, count / 2, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        rc = (int)e;
    }
    if (truth && rc == 0) std::memcpy(truth, tr.data(), sizeof(double) * 3 * count);
    cudaFree(ev);
    cudaFree(mev);
    return rc;
}

}  // extern "C"
