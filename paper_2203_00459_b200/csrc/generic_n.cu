// generic_n.cu — rotation stage for grid sides that are not powers of two
// (the reference's own sizes are odd, matcher.cpp:25 / geometry.cpp:38).
//
// The magnitude spectrum must be the N-point DFT of the reference
// (spectral.cpp:73-117), so rows and columns use Bluestein's chirp-z
// identity on top of the power-of-two register FFT (fft.cuh):
//   X[k] = w[k] sum_n (x[n] w[n]) conj(w[k - n]),  w[n] = exp(-i pi n^2 / N),
// a circular convolution of length L >= 2N - 1 done as FFT_L, a product with
// the precomputed FFT_L of the kernel b[m] = conj(w[m]) (|m| < N, scaled by
// 1/L) and an inverse FFT_L. Everything else (band, polar gather, angular
// correlation, translation stage) runs on the common kernels; the
// translation stage embeds the scans in a power-of-two grid.
#include <cuda_runtime.h>

#include "fft.cuh"
#include "pipeline.h"

namespace fscan_detail {
namespace {

using fscan_fft::cadd;
using fscan_fft::cconj;
using fscan_fft::cmul;
using fscan_fft::csub;
using fscan_fft::fft_regs;
using fscan_fft::Lay;

constexpr int kBsRowThreads = 128;

// K1a (any N): rows of f~ = f*mf, g~ = g*mg (written zero-embedded in the
// np x np translation buffers), Hann window, packed row DFT of f~w + i g~w
// into zbuf [pair][N][N].
template <int L>
__global__ void __launch_bounds__(kBsRowThreads) k_rot_rows_bs(Params p) {
    constexpr int T = L / 16;
    constexpr int PER = kBsRowThreads / T > 0 ? kBsRowThreads / T : 1;  // rows per CTA
    constexpr int STRIDE = L + 2;                                      // float2 per transform buffer
    extern __shared__ float smem[];
    const int n = p.n, np = p.np, pair = blockIdx.y;
    const int tr = threadIdx.x / T, t = threadIdx.x % T;
    const int y = blockIdx.x * PER + tr;
    const bool row_ok = tr < PER && y < n;
    const Lay<1> lay{reinterpret_cast<float2*>(smem) + tr * STRIDE, 0};
    const size_t yy = (size_t)(row_ok ? y : 0);
    // the two real grids of this transform: scans `pair` of f and g, or in chain
    // mode (odometry) scans 2*pair and 2*pair+1 of one sequence (the last one
    // duplicated for an odd count) with their masked copies stored per scan
    const float *fp, *gp, *mfp = nullptr, *mgp = nullptr;
    float *ftp, *gtp;
    size_t fi = pair, gi = pair;
    if (p.chain) {
        fi = 2 * (size_t)pair;
        gi = (size_t)min(2 * pair + 1, p.n_scans - 1);
        fp = p.f + fi * n * n + yy * n;
        gp = p.f + gi * n * n + yy * n;
        if (p.mf) {
            mfp = p.mf + fi * n * n + yy * n;
            mgp = p.mf + gi * n * n + yy * n;
        }
        ftp = p.ft + fi * np * np + yy * np;
        gtp = p.ft + gi * np * np + yy * np;
    } else {
        fp = p.f + ((size_t)pair * n + yy) * n;
        gp = p.g + ((size_t)pair * n + yy) * n;
        if (p.mf) {
            mfp = p.mf + ((size_t)pair * n + yy) * n;
            mgp = p.mg + ((size_t)pair * n + yy) * n;
        }
        ftp = p.ft + (size_t)pair * np * np + yy * np;
        gtp = p.gt + (size_t)pair * np * np + yy * np;
    }
    const float hy = p.hann[yy];
    int badf = 0, badg = 0;
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int x = t + m * T;
        float2 a = make_float2(0.f, 0.f);
        if (row_ok && x < n) {
            float fv = __ldg(fp + x), gv = __ldg(gp + x);
            if (mfp) {
                const float ma = __ldg(mfp + x), mb = __ldg(mgp + x);
                if (!(ma >= 0.0f && ma <= 1.0f)) badf |= 2;
                if (!(mb >= 0.0f && mb <= 1.0f)) badg |= 2;
                fv *= ma;
                gv *= mb;
            }
            if (!isfinite(fv)) badf |= 1;
            if (!isfinite(gv)) badg |= 1;
            ftp[x] = fv;
            gtp[x] = gv;
            const float w = hy * __ldg(p.hann + x);
            a = cmul(make_float2(fv * w, gv * w), __ldg(p.bs_chirp + x));
        }
        v[m] = a;
    }
    fft_regs<L, -1, (T <= 32)>(v, t, lay, p.tw_L);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = cmul(v[m], __ldg(p.bs_kern + t + m * T));
    fft_regs<L, +1, (T <= 32)>(v, t, lay, p.tw_L);
    if (row_ok) {
        float2* z = p.zbuf + ((size_t)pair * n + y) * n;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int k = t + m * T;
            if (k < n) z[k] = cmul(v[m], __ldg(p.bs_chirp + k));
        }
    }
    if (p.chain) {  // flags per scan of the sequence
        if (badf) atomicOr(p.flags + fi, badf);
        if (badg) atomicOr(p.flags + gi, badg);
    } else if (badf | badg) {
        atomicOr(p.flags + pair, badf | badg);
    }
}

// K1b (any N): 4 output columns u0..u0+3 and their mirrors (N - u) mod N as 8
// interleaved column DFTs; F = (Z[v,u] + conj Z[-v,-u]) / 2, G = (Z - conj Z)/2i,
// |F|, |G| times the band on the half plane u < W, into the (|F|,|G|) tiles.
template <int L>
__global__ void __launch_bounds__(8 * (L / 16)) k_rot_cols_bs(Params p) {
    constexpr int T = L / 16;
    extern __shared__ float smem[];
    const int n = p.n, W = p.nw, pair = blockIdx.y;
    const int u0 = blockIdx.x * 4;
    const int c = threadIdx.x % 8, t = threadIdx.x / 8;
    const int u = u0 + (c & 3);
    const int col = c < 4 ? (u % n) : ((n - u) % n);
    const bool col_ok = u < W;
    float2* sbuf = reinterpret_cast<float2*>(smem);
    const Lay<8> lay{sbuf, c};
    const float2* z = p.zbuf + (size_t)pair * n * n;
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int r = t + m * T;
        v[m] = (col_ok && r < n) ? cmul(z[(size_t)r * n + col], __ldg(p.bs_chirp + r)) : make_float2(0.f, 0.f);
    }
    fft_regs<L, -1>(v, t, lay, p.tw_L);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = cmul(v[m], __ldg(p.bs_kern + t + m * T));
    fft_regs<L, +1>(v, t, lay, p.tw_L);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int k = t + m * T;
        if (k < n) lay.put(k, cmul(v[m], __ldg(p.bs_chirp + k)));
    }
    __syncthreads();
    const int cn = n / 2;
    float2* out = reinterpret_cast<float2*>(p.mag) + (size_t)pair * p.mag_plane;
    for (int o = threadIdx.x; o < n * 4; o += blockDim.x) {
        const int cc = o & 3, vc = o >> 2;
        const int uu = u0 + cc;
        if (uu >= W) continue;
        const int vn = (vc - cn + n) % n;  // natural row of centred row vc
        const int vm = (n - vn) % n;       // row of -v
        const float2 z1 = Lay<8>{sbuf, cc}.get(vn);
        const float2 z2 = Lay<8>{sbuf, 4 + cc}.get(vm);
        const float fr = z1.x + z2.x, fi = z1.y - z2.y;  // Z1 + conj(Z2)
        const float gr = z1.x - z2.x, gi = z1.y + z2.y;  // Z1 - conj(Z2)
        const int2 bd = __ldg(p.band + vc);
        const bool in = (uu >= bd.x) && (uu <= bd.y);
        out[((size_t)(uu >> 3) * n + vc) * 8 + (uu & 7)] =
            in ? make_float2(0.5f * sqrtf(fr * fr + fi * fi), 0.5f * sqrtf(gr * gr + gi * gi)) : make_float2(0.f, 0.f);
    }
}

template <typename K>
cudaError_t set_smem_bs(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return cudaSuccess;
}

template <int L>
cudaError_t rows_bs(const Params& p, cudaStream_t s) {
    constexpr int T = L / 16;
    constexpr int PER = kBsRowThreads / T > 0 ? kBsRowThreads / T : 1;
    const int threads = PER * T;
    const size_t sm = (size_t)PER * (L + 2) * sizeof(float2);
    cudaError_t e = set_smem_bs(k_rot_rows_bs<L>, sm);
    if (e != cudaSuccess) return e;
    k_rot_rows_bs<L><<<dim3((p.n + PER - 1) / PER, p.batch), threads, sm, s>>>(p);
    return cudaGetLastError();
}

template <int L>
cudaError_t cols_bs(const Params& p, cudaStream_t s) {
    const size_t sm = (size_t)fscan_fft::part_floats<L, 8>() * sizeof(float);
    cudaError_t e = set_smem_bs(k_rot_cols_bs<L>, sm);
    if (e != cudaSuccess) return e;
    k_rot_cols_bs<L><<<dim3((p.zcols + 3) / 4, p.batch), 8 * (L / 16), sm, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

#define FSCAN_DISPATCH_L(FN)                      \
    switch (p.bs_L) {                             \
        case 128: return FN<128>(p, s);           \
        case 256: return FN<256>(p, s);           \
        case 512: return FN<512>(p, s);           \
        case 1024: return FN<1024>(p, s);         \
        case 2048: return FN<2048>(p, s);         \
        default: return cudaErrorInvalidValue;    \
    }

cudaError_t launch_rot_rows_bs(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_L(rows_bs) }
cudaError_t launch_rot_cols_bs(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_L(cols_bs) }

}  // namespace fscan_detail
