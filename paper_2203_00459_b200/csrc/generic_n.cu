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
            in ? make_float2(0.5f * fscan_fft::sqrt_fast(fr * fr + fi * fi), 0.5f * fscan_fft::sqrt_fast(gr * gr + gi * gi)) : make_float2(0.f, 0.f);
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


// ---------------------------------------------------------------- N = 255
// The reference's default grid (matcher.hpp:13-26: n_xy = 255) gets an exact
// prime-factor DFT instead of Bluestein: 255 = 15 * 17 (coprime), so by the
// Good-Thomas map n = (17 n1 + 15 n2) mod 255, k = (136 k1 + 120 k2) mod 255
// (136 = 17 * (17^-1 mod 15), 120 = 15 * (15^-1 mod 17)) the DFT is 15
// 17-point DFTs over n2 followed by 17 15-point DFTs over n1 with no twiddles
// (15 = 3 * 5 by the same map: n1 = (5a + 3b) mod 15, k1 = (10c + 6d) mod 15).
// The small DFTs are straight-line code with compile-time constants: ~31 flops
// per point against ~180 for the two length-512 Bluestein transforms.
constexpr int kPfaN = 255;

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }

// 3-point DFT, SIGN = -1 forward / +1 inverse (unnormalised)
template <int SIGN>
__device__ __forceinline__ void dft3(float2& x0, float2& x1, float2& x2) {
    constexpr float h = 8.660254038e-01f;  // sqrt(3)/2
    const float2 t1 = cadd(x1, x2), t2 = csub(x1, x2);
    const float2 m = f2(fmaf(-0.5f, t1.x, x0.x), fmaf(-0.5f, t1.y, x0.y));
    x0 = cadd(x0, t1);
    // X1 = m + SIGN * i * h * t2, X2 = m - SIGN * i * h * t2
    const float2 r = SIGN < 0 ? f2(h * t2.y, -h * t2.x) : f2(-h * t2.y, h * t2.x);
    x1 = cadd(m, r);
    x2 = csub(m, r);
}

// 5-point DFT
template <int SIGN>
__device__ __forceinline__ void dft5(float2& x0, float2& x1, float2& x2, float2& x3, float2& x4) {
    constexpr float c1 = 3.090169944e-01f, c2 = -8.090169944e-01f;  // cos(2 pi / 5), cos(4 pi / 5)
    constexpr float s1 = 9.510565163e-01f, s2 = 5.877852523e-01f;   // sin(2 pi / 5), sin(4 pi / 5)
    const float2 t1 = cadd(x1, x4), t2 = cadd(x2, x3), t3 = csub(x1, x4), t4 = csub(x2, x3);
    const float2 a1 = f2(fmaf(c2, t2.x, fmaf(c1, t1.x, x0.x)), fmaf(c2, t2.y, fmaf(c1, t1.y, x0.y)));
    const float2 a2 = f2(fmaf(c1, t2.x, fmaf(c2, t1.x, x0.x)), fmaf(c1, t2.y, fmaf(c2, t1.y, x0.y)));
    const float2 b1 = f2(fmaf(s2, t4.x, s1 * t3.x), fmaf(s2, t4.y, s1 * t3.y));
    const float2 b2 = f2(fmaf(-s1, t4.x, s2 * t3.x), fmaf(-s1, t4.y, s2 * t3.y));
    x0 = cadd(x0, cadd(t1, t2));
    // forward: X1 = a1 - i b1, X4 = a1 + i b1, X2 = a2 - i b2, X3 = a2 + i b2
    const float2 r1 = SIGN < 0 ? f2(b1.y, -b1.x) : f2(-b1.y, b1.x);
    const float2 r2 = SIGN < 0 ? f2(b2.y, -b2.x) : f2(-b2.y, b2.x);
    x1 = cadd(a1, r1);
    x4 = csub(a1, r1);
    x2 = cadd(a2, r2);
    x3 = csub(a2, r2);
}

// 15-point DFT (natural order in and out) as 3 x 5 prime factor
template <int SIGN>
__device__ __forceinline__ void dft15(float2 (&x)[15]) {
    float2 t[3][5];
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        float2 u0 = x[(3 * b) % 15], u1 = x[(5 + 3 * b) % 15], u2 = x[(10 + 3 * b) % 15];
        dft3<SIGN>(u0, u1, u2);
        t[0][b] = u0;
        t[1][b] = u1;
        t[2][b] = u2;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dft5<SIGN>(t[c][0], t[c][1], t[c][2], t[c][3], t[c][4]);
#pragma unroll
        for (int d = 0; d < 5; ++d) x[(10 * c + 6 * d) % 15] = t[c][d];
    }
}

// 17-point DFT (natural order in and out), symmetric form:
// X[k] = x0 + sum_j (x_j + x_{17-j}) cos(2 pi jk/17) -/+ i (x_j - x_{17-j}) sin(2 pi jk/17)
template <int SIGN>
__device__ __forceinline__ void dft17(float2 (&x)[17]) {
    constexpr float C[9] = {1.000000000e+00f, 9.324722294e-01f, 7.390089172e-01f, 4.457383558e-01f, 9.226835946e-02f,
                            -2.736629901e-01f, -6.026346364e-01f, -8.502171357e-01f, -9.829730997e-01f};
    constexpr float S[9] = {0.000000000e+00f, 3.612416662e-01f, 6.736956436e-01f, 8.951632914e-01f, 9.957341763e-01f,
                            9.618256432e-01f, 7.980172273e-01f, 5.264321629e-01f, 1.837495178e-01f};
    float2 a[8], b[8];
#pragma unroll
    for (int j = 1; j <= 8; ++j) {
        a[j - 1] = cadd(x[j], x[17 - j]);
        b[j - 1] = csub(x[j], x[17 - j]);
    }
    const float2 x0 = x[0];
    float2 s0 = x0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s0 = cadd(s0, a[j]);
    x[0] = s0;
#pragma unroll
    for (int k = 1; k <= 8; ++k) {
        float ax = x0.x, ay = x0.y, bx = 0.f, by = 0.f;
#pragma unroll
        for (int j = 1; j <= 8; ++j) {
            const int m = (j * k) % 17;
            const float cm = m <= 8 ? C[m] : C[17 - m];
            const float sm = m <= 8 ? S[m] : -S[17 - m];
            ax = fmaf(cm, a[j - 1].x, ax);
            ay = fmaf(cm, a[j - 1].y, ay);
            bx = fmaf(sm, b[j - 1].y, bx);
            by = fmaf(sm, b[j - 1].x, by);
        }
        // forward: X[k] = (ax + bx, ay - by), X[17 - k] = (ax - bx, ay + by)
        if (SIGN < 0) {
            x[k] = f2(ax + bx, ay - by);
            x[17 - k] = f2(ax - bx, ay + by);
        } else {
            x[k] = f2(ax - bx, ay + by);
            x[17 - k] = f2(ax + bx, ay - by);
        }
    }
}

// One 255-point DFT per 17 threads (slot s of transform buffer `buf`, natural
// order in and out, in place). Every thread of the CTA must call it (it holds
// __syncthreads); `live` masks the threads outside a transform.
template <int SIGN>
__device__ __forceinline__ void dft255_smem(float2* buf, int s, bool live) {
    if (live && s < 15) {  // 15 17-point DFTs over n2 for n1 = s, in place
        float2 x[17];
        const int base = 17 * s;
#pragma unroll
        for (int n2 = 0; n2 < 17; ++n2) {
            int i = base + 15 * n2;
            i -= i >= kPfaN ? kPfaN : 0;
            x[n2] = buf[i];
        }
        dft17<SIGN>(x);
#pragma unroll
        for (int n2 = 0; n2 < 17; ++n2) {
            int i = base + 15 * n2;
            i -= i >= kPfaN ? kPfaN : 0;
            buf[i] = x[n2];
        }
    }
    __syncthreads();
    float2 y[15];
    if (live) {  // 17 15-point DFTs over n1 for k2 = s
        const int base = 15 * s;
#pragma unroll
        for (int n1 = 0; n1 < 15; ++n1) {
            int i = base + 17 * n1;
            i -= i >= kPfaN ? kPfaN : 0;
            y[n1] = buf[i];
        }
        dft15<SIGN>(y);
    }
    __syncthreads();
    if (live) {  // X[(136 k1 + 120 s) mod 255]
        int i = (120 * s) % kPfaN;
#pragma unroll
        for (int k1 = 0; k1 < 15; ++k1) {
            buf[i] = y[k1];
            i += 136;
            i -= i >= kPfaN ? kPfaN : 0;
        }
    }
    __syncthreads();
}

constexpr int kPfaRows = 15;         // K1a: rows per CTA (17 CTAs per pair)
constexpr int kPfaSP = kPfaN + 2;    // float2 per transform buffer (odd: rows on distinct banks)
constexpr int kPfaRowThreads = 256;  // 15 transforms x 17 slots (+1 idle)

// K1a, N = 255: as k_rot_rows_bs with the prime-factor DFT; stores only the
// columns K1b reads (k < zcols and their mirrors k > N - zcols).
__global__ void __launch_bounds__(kPfaRowThreads) k_rot_rows_pfa255(Params p) {
    __shared__ float2 buf[kPfaRows * kPfaSP];
    constexpr int n = kPfaN;
    const int np = p.np, pair = blockIdx.y, y0 = blockIdx.x * kPfaRows;
    const int x = threadIdx.x;
    const bool xin = x < n;
    const float hx = xin ? __ldg(p.hann + x) : 0.f;
    int badf = 0, badg = 0;
    size_t fi = pair, gi = pair;
    if (p.chain) {
        fi = 2 * (size_t)pair;
        gi = (size_t)min(2 * pair + 1, p.n_scans - 1);
    }
    // five rows per round with every load issued before any use (the stores of
    // f~, g~ could alias the inputs for the compiler, so it would not hoist them)
    constexpr int RB = 5;
#pragma unroll 1
    for (int r0 = 0; r0 < kPfaRows; r0 += RB) {
        float fv[RB], gv[RB], ma[RB], mb[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int y = y0 + r0 + i;
            const size_t fo = (p.chain ? fi * n + y : (size_t)pair * n + y) * n + x;
            const size_t go = (p.chain ? gi * n + y : (size_t)pair * n + y) * n + x;
            const float* gsrc = p.chain ? p.f : p.g;
            const float* mgsrc = p.chain ? p.mf : p.mg;
            fv[i] = xin ? __ldg(p.f + fo) : 0.f;
            gv[i] = xin ? __ldg(gsrc + go) : 0.f;
            ma[i] = (xin && p.mf) ? __ldg(p.mf + fo) : 1.f;
            mb[i] = (xin && p.mf) ? __ldg(mgsrc + go) : 1.f;
        }
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int y = y0 + r0 + i;
            if (!xin) continue;
            float a = fv[i], b = gv[i];
            if (p.mf) {
                if (!(ma[i] >= 0.0f && ma[i] <= 1.0f)) badf |= 2;
                if (!(mb[i] >= 0.0f && mb[i] <= 1.0f)) badg |= 2;
                a *= ma[i];
                b *= mb[i];
            }
            if (!isfinite(a)) badf |= 1;
            if (!isfinite(b)) badg |= 1;
            float* ftp = p.ft + (p.chain ? fi : (size_t)pair) * np * np + (size_t)y * np;
            float* gtp = (p.chain ? p.ft + gi * np * np : p.gt + (size_t)pair * np * np) + (size_t)y * np;
            ftp[x] = a;
            gtp[x] = b;
            const float w = __ldg(p.hann + y) * hx;
            buf[(r0 + i) * kPfaSP + x] = f2(a * w, b * w);
        }
    }
    __syncthreads();
    const int tr = threadIdx.x / 17, s = threadIdx.x % 17;
    const bool live = tr < kPfaRows;
    dft255_smem<-1>(buf + (live ? tr : 0) * kPfaSP, s, live);
    // the columns K1b reads, coalesced per row
    const int zc = p.zcols;
#pragma unroll 3
    for (int r = 0; r < kPfaRows; ++r)
        if (xin && (x < zc || x > n - zc)) p.zbuf[((size_t)pair * n + y0 + r) * n + x] = buf[r * kPfaSP + x];
    if (p.chain) {
        if (badf) atomicOr(p.flags + fi, badf);
        if (badg) atomicOr(p.flags + gi, badg);
    } else if (badf | badg) {
        atomicOr(p.flags + pair, badf | badg);
    }
}

constexpr int kPfaCSP = kPfaN + 2;    // K1b buffer stride: the 16 columns of a row on distinct banks
constexpr int kPfaColThreads = 288;  // 16 transforms (8 columns u, 8 mirrors) x 17 slots

// K1b, N = 255: 8 columns u0..u0+7 and their mirrors (N - u) mod N, F/G
// separation, |F|, |G| times the band into the (|F|,|G|) tiles (as k_rot_cols_bs).
__global__ void __launch_bounds__(kPfaColThreads) k_rot_cols_pfa255(Params p) {
    __shared__ float2 buf[16 * kPfaCSP];
    constexpr int n = kPfaN;
    const int W = p.nw, pair = blockIdx.y, u0 = blockIdx.x * 8;
    const int ulim = min(W, p.zcols);
    const float2* z = p.zbuf + (size_t)pair * n * n;
    constexpr int U = 5;  // loads in flight per thread
#pragma unroll 1
    for (int e0 = threadIdx.x; e0 < n * 16; e0 += U * kPfaColThreads) {
        float2 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int e = e0 + k * kPfaColThreads;
            const int row = e >> 4, c = e & 15;
            const int u = u0 + (c & 7);
            const int col = c < 8 ? u : (n - u) % n;
            v[k] = (e < n * 16 && u < ulim) ? z[(size_t)row * n + col] : f2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int e = e0 + k * kPfaColThreads;
            if (e < n * 16) buf[(e & 15) * kPfaCSP + (e >> 4)] = v[k];
        }
    }
    __syncthreads();
    const int tr = threadIdx.x / 17, s = threadIdx.x % 17;
    const bool live = tr < 16;
    dft255_smem<-1>(buf + (live ? tr : 0) * kPfaCSP, s, live);
    const int cn = n / 2;
    float2* out = reinterpret_cast<float2*>(p.mag) + (size_t)pair * p.mag_plane;
    for (int o = threadIdx.x; o < n * 8; o += kPfaColThreads) {
        const int cc = o & 7, vc = o >> 3;
        const int uu = u0 + cc;
        if (uu >= W) continue;
        const int vn = (vc - cn + n) % n;  // natural row of centred row vc
        const int vm = (n - vn) % n;       // row of -v
        const float2 z1 = buf[cc * kPfaCSP + vn];
        const float2 z2 = buf[(8 + cc) * kPfaCSP + vm];
        const float fr = z1.x + z2.x, fi = z1.y - z2.y;  // Z1 + conj(Z2)
        const float gr = z1.x - z2.x, gi = z1.y + z2.y;  // Z1 - conj(Z2)
        const int2 bd = __ldg(p.band + vc);
        const bool in = (uu >= bd.x) && (uu <= bd.y);
        out[((size_t)(uu >> 3) * n + vc) * 8 + (uu & 7)] =
            in ? make_float2(0.5f * fscan_fft::sqrt_fast(fr * fr + fi * fi), 0.5f * fscan_fft::sqrt_fast(gr * gr + gi * gi)) : make_float2(0.f, 0.f);
    }
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

cudaError_t launch_rot_rows_bs(const Params& p, cudaStream_t s) {
    if (p.n == kPfaN) {
        k_rot_rows_pfa255<<<dim3(kPfaN / kPfaRows, p.batch), kPfaRowThreads, 0, s>>>(p);
        return cudaGetLastError();
    }
    FSCAN_DISPATCH_L(rows_bs)
}
cudaError_t launch_rot_cols_bs(const Params& p, cudaStream_t s) {
    if (p.n == kPfaN) {
        k_rot_cols_pfa255<<<dim3((p.zcols + 7) / 8, p.batch), kPfaColThreads, 0, s>>>(p);
        return cudaGetLastError();
    }
    FSCAN_DISPATCH_L(cols_bs)
}

}  // namespace fscan_detail
