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

#include "synth_scene.h"

using fsynth::PairScene;
using fsynth::build_scene;
using fsynth::sequence_scan;

namespace {

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
