// Micro-benchmark (dev tool, not product): the one data exchange of a 256-point
// radix-16 x 16 FFT (fft.cuh) through shared memory (the product's layout,
// Geom<256>) versus a warp-shuffle transpose (4 xor-butterfly rounds over the
// 16 lanes of a transform), everything else identical (registers, dft16,
// global twiddle table). Each thread block runs ITERS forward+inverse pairs
// per transform on register-resident data; prints one JSON line with the time
// per 256-point transform of each variant and the max |difference| of their
// results. Build: see tools/microbench/run.sh.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "fft.cuh"

using namespace fscan_fft;

constexpr int K = 256, T = 16, THREADS = 256, ITERS = 64;
using G = Geom<K, THREADS>;

// 16x16 transpose across the 16 lanes of a transform: lane l ends with the
// elements r = l of every lane (xor butterflies of 8, 4, 2, 1 lanes)
__device__ __forceinline__ void shfl_transpose16(float2 (&v)[16], int lane) {
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
        const bool hi = lane & s;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            if (r & s) continue;
            const float2 send = hi ? v[r] : v[r | s];
            float2 recv;
            recv.x = __shfl_xor_sync(0xffffffffu, send.x, s);
            recv.y = __shfl_xor_sync(0xffffffffu, send.y, s);
            if (hi)
                v[r] = recv;
            else
                v[r | s] = recv;
        }
    }
}

template <int SIGN>
__device__ __forceinline__ void fft256_shfl(float2 (&v)[16], int t, const float2* __restrict__ tw) {
    dft16<SIGN>(v);           // stage 1 (span 1, no twiddles): y[16 t + r] held as v[r]
    shfl_transpose16(v, t);   // thread t now holds y[t + 16 m] as v[m]
    // stage 2 exactly as fft_regs runs it (the last stage never touches the buffer)
    stage<K, 16, 16, true, SIGN, true>(v, t, Lay<1>{nullptr, 0}, tw);
}

template <bool SHFL>
__global__ void __launch_bounds__(THREADS) k_bench(const float2* __restrict__ in, float2* __restrict__ out,
                                                     const float2* __restrict__ tw) {
    extern __shared__ float smem[];
    int tr, t;
    G::map(threadIdx.x, tr, t);
    const int gtr = blockIdx.x * G::PER_CTA + tr;
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = in[(size_t)gtr * K + t + m * T];
    const auto lay = G::lay(smem, tr);
    for (int it = 0; it < ITERS; ++it) {
        if constexpr (SHFL) {
            fft256_shfl<-1>(v, t, tw);
            fft256_shfl<+1>(v, t, tw);
        } else {
            fft_regs<K, -1, true>(v, t, lay, tw);
            fft_regs<K, +1, true>(v, t, lay, tw);
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = make_float2(v[m].x * (1.0f / K), v[m].y * (1.0f / K));
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) out[(size_t)gtr * K + t + m * T] = v[m];
}

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e = (x);                                                                       \
        if (e != cudaSuccess) {                                                                    \
            printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__);              \
            return 1;                                                                              \
        }                                                                                          \
    } while (0)

int main() {
    const int blocks = 148 * 8, ntr = blocks * G::PER_CTA;
    std::vector<float2> h((size_t)ntr * K), tw(K);
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_float2(std::sin(0.001 * i), std::cos(0.0007 * i));
    for (int k = 0; k < K; ++k) tw[k] = make_float2((float)std::cos(-2 * M_PI * k / K), (float)std::sin(-2 * M_PI * k / K));
    float2 *d_in, *d_a, *d_b, *d_tw;
    CK(cudaMalloc(&d_in, h.size() * 8));
    CK(cudaMalloc(&d_a, h.size() * 8));
    CK(cudaMalloc(&d_b, h.size() * 8));
    CK(cudaMalloc(&d_tw, K * 8));
    CK(cudaMemcpy(d_in, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_tw, tw.data(), K * 8, cudaMemcpyHostToDevice));
    const size_t sm = (size_t)G::FLOATS * 4;
    CK(cudaFuncSetAttribute(k_bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms[2] = {0, 0};
    for (int rep = 0; rep < 3; ++rep)
        for (int v = 0; v < 2; ++v) {
            cudaEventRecord(e0);
            if (v == 0)
                k_bench<false><<<blocks, THREADS, sm>>>(d_in, d_a, d_tw);
            else
                k_bench<true><<<blocks, THREADS, 0>>>(d_in, d_b, d_tw);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            if (rep > 0) ms[v] += t / 2;
        }
    std::vector<float2> a(h.size()), b(h.size());
    CK(cudaMemcpy(a.data(), d_a, a.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), d_b, b.size() * 8, cudaMemcpyDeviceToHost));
    double md = 0, mx = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        md = std::fmax(md, std::fabs(a[i].x - b[i].x) + std::fabs(a[i].y - b[i].y));
        mx = std::fmax(mx, std::fabs(a[i].x) + std::fabs(a[i].y));
    }
    const double n_fft = (double)ntr * ITERS * 2;
    printf("{\"bench\": \"256-point radix-16x16 FFT exchange: shared memory vs warp shuffle\", "
           "\"transforms\": %.0f, \"smem_ns_per_fft\": %.4f, \"shfl_ns_per_fft\": %.4f, "
           "\"shfl_over_smem\": %.3f, \"max_abs_diff\": %.3e, \"max_abs\": %.3e, \"smem_bytes_per_cta\": %zu}\n",
           n_fft, ms[0] * 1e6 / n_fft, ms[1] * 1e6 / n_fft, ms[1] / ms[0], md, mx, sm);
    return 0;
}
