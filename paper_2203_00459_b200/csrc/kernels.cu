// kernels.cu — sm_100a kernels of the decoupled Fourier pose search.
//
// Pipeline per batch of pairs, all fp32 SIMT (no dense
// contraction, so no tensor cores), FFTs from fft.cuh:
//   K0 polar_to_cart  raw polar sweep -> Cartesian grid            (config 3; no reference)
//   K1a rot_rows      mask, finiteness, Hann, packed row FFTs       matcher.cpp:113-118, imageops.cpp:130-137
//   K1b rot_cols      column FFTs, split f/g, |F|, band-pass        spectral.cpp:73-117, matcher.cpp:120-126
//   K2  rot_polar     polar gather, radial sums, angular xcorr,
//                     hard + soft argmax over theta                 matcher.cpp:128-153, imageops.cpp:81-113
//   K3  xlat_rows     de-rotation of g, packed row FFTs (2N)        imageops.cpp:61-79,115-124, spectral.cpp:126-131
//   K4  xlat_cols     column FFTs (2N), conj(F) G, inverse columns  spectral.cpp:131-136
//   K5  xlat_out      inverse rows (C2R), crop/flip, block argmax   spectral.cpp:137-151, matcher.cpp:171-182
//   K6  finalize      global argmax, soft argmax, back-rotation     matcher.cpp:184-208
// The zero padding to P = 2N of the translation stage is never materialised:
// both scans are placed at offset 0 (a common shift cancels in conj(F) G) and
// each 2N-point transform of a half-zero signal is two N-point transforms
// (even outputs: FFT_N(x); odd outputs: FFT_N(x * W_2N^n)).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft.cuh"
#include "pipeline.h"
#include "polar.h"

namespace fscan_detail {

using fscan_fft::Cfg;
using fscan_fft::cadd;
using fscan_fft::cconj;
using fscan_fft::cmul;
using fscan_fft::csub;
using fscan_fft::fft_regs;
using fscan_fft::spad;

namespace {

constexpr int kRowThreads = 256;

template <int N>
__host__ __device__ constexpr int rows_per_block() {
    return kRowThreads / (N / 16) < 1 ? 1 : kRowThreads / (N / 16);
}

__device__ __forceinline__ float bilerp(float fr, float fc, float a00, float a01, float a10, float a11) {
    // sample_bilinear (imageops.cpp:24-25) operation order, fp32
    return (1.0f - fr) * ((1.0f - fc) * a00 + fc * a01) + fr * ((1.0f - fc) * a10 + fc * a11);
}

// ---------------------------------------------------------------- K1a
// rows of f~ = f*mf and g~ = g*mg: write the masked scans (translation stage
// input), window by the separable Hann w[r]*w[c], FFT the packed row
// z = f~w + i g~w.
template <int N>
__global__ void __launch_bounds__(kRowThreads) k_rot_rows(Params p) {
    constexpr int T = N / 16;
    constexpr int RPB = rows_per_block<N>();
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    const int tr = threadIdx.x / T, t = threadIdx.x % T;
    const int y = blockIdx.x * RPB + tr;
    float* sb = smem + tr * Cfg<N>::kFloats;
    const size_t base = ((size_t)pair * N + y) * N;
    const float hy = p.hann[y];
    int bad = 0;
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int x = t + m * T;
        float fv = __ldg(p.f + base + x);
        float gv = __ldg(p.g + base + x);
        if (p.mf) {
            const float a = __ldg(p.mf + base + x), b = __ldg(p.mg + base + x);
            if (!(a >= 0.0f && a <= 1.0f) || !(b >= 0.0f && b <= 1.0f)) bad |= 2;
            fv *= a;
            gv *= b;
        }
        if (!isfinite(fv) || !isfinite(gv)) bad |= 1;
        p.ft[base + x] = fv;
        p.gt[base + x] = gv;
        const float w = hy * __ldg(p.hann + x);
        v[m] = make_float2(fv * w, gv * w);
    }
    fft_regs<N, -1>(v, t, sb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) p.zbuf[base + t + m * T] = v[m];
    if (bad) atomicOr(p.flags + pair, bad);
}

// ---------------------------------------------------------------- K1b
// 8 output columns u in [u0, u0+8) plus their mirrors (N-u) mod N; column
// FFTs; F = (Z[v,u] + conj Z[-v,-u]) / 2, G = (Z[v,u] - conj Z[-v,-u]) / 2i;
// |F|, |G| times the annular band, written as an [N centred rows][8] tile.
template <int N>
__global__ void __launch_bounds__(N) k_rot_cols(Params p) {
    constexpr int T = N / 16;
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    const int u0 = blockIdx.x * 8;
    const int c = threadIdx.x % 16, t = threadIdx.x / 16;
    const int col = c < 8 ? (u0 + c) : ((N - (u0 + c - 8)) & (N - 1));
    float* sb = smem + c * Cfg<N>::kFloats;
    const float2* z = p.zbuf + (size_t)pair * N * N;
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = z[(size_t)(t + m * T) * N + col];
    fft_regs<N, -1>(v, t, sb, p.tw_n);
    float* sre = sb;
    float* sim = sb + Cfg<N>::kHalf;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int q = spad(t + m * T);
        sre[q] = v[m].x;
        sim[q] = v[m].y;
    }
    __syncthreads();
    float* outf = p.mag + (((size_t)pair * 2 + 0) * (N / 16) + blockIdx.x) * (size_t)(N * 8);
    float* outg = p.mag + (((size_t)pair * 2 + 1) * (N / 16) + blockIdx.x) * (size_t)(N * 8);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int o = threadIdx.x + q * N;  // o = v_c * 8 + cc
        const int cc = o & 7, vc = o >> 3;
        const int vn = (vc + N / 2) & (N - 1);  // natural row of centred row vc
        const int vm = (N - vn) & (N - 1);      // row of -v
        const float* a = smem + cc * Cfg<N>::kFloats;
        const float* b = smem + (8 + cc) * Cfg<N>::kFloats;
        const float2 z1 = make_float2(a[spad(vn)], a[Cfg<N>::kHalf + spad(vn)]);
        const float2 z2 = make_float2(b[spad(vm)], b[Cfg<N>::kHalf + spad(vm)]);
        const float fr = z1.x + z2.x, fi = z1.y - z2.y;  // Z1 + conj(Z2)
        const float gr = z1.x - z2.x, gi = z1.y + z2.y;  // Z1 - conj(Z2)
        const int2 bd = __ldg(p.band + vc);
        const int u = u0 + cc;
        const bool in = (u >= bd.x) && (u <= bd.y);
        outf[o] = in ? 0.5f * sqrtf(fr * fr + fi * fi) : 0.0f;
        outg[o] = in ? 0.5f * sqrtf(gr * gr + gi * gi) : 0.0f;
    }
}

// ---------------------------------------------------------------- K2
constexpr int kPolarThreads = 512;

__device__ __forceinline__ float tile_at(const float* m, int n, int r, int u) {
    return __ldg(m + ((size_t)(u >> 3) * n + r) * 8 + (u & 7));
}

__global__ void __launch_bounds__(kPolarThreads) k_rot_polar(Params p) {
    extern __shared__ double dsm[];
    const int pair = blockIdx.x;
    const int nt = p.n_theta, L = p.L, pad = p.pad, n = p.n;
    double* A = dsm;           // wrap-extended radial-sum profiles, length L
    double* B = dsm + L;
    double* s = dsm + 2 * L;   // theta surface, n_theta
    double* red_v = s + nt;    // block reduction scratch (32 entries each)
    int* red_i = (int*)(red_v + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = kPolarThreads / 32;
    RotState* rs = p.rot + pair;

    if (nt == 1) {  // matcher.cpp:103-110
        if (threadIdx.x == 0) {
            rs->theta = 0.0;
            rs->st = 0.0;
            rs->ct = 1.0;
            rs->peak = 0.0;
            rs->hard = 0.0;
            rs->bin = 0;
            rs->identity = 1;
            if (p.theta_surf) p.theta_surf[pair] = 0.0;
            if (p.theta_only) p.theta_only[pair] = 0.0;
        }
        return;
    }

    const float* mf = p.mag + (size_t)pair * 2 * n * (n / 2);
    const float* mg = mf + (size_t)n * (n / 2);
    // radial sums of the bilinear polar resample (cart2pol) of |F| and |G|
    for (int i = warp; i < nt; i += nwarps) {
        double af = 0.0, ag = 0.0;
        const PolarTap* row = p.taps + (size_t)i * p.n_live;
        for (int jj = lane; jj < p.n_live; jj += 32) {
            const PolarTap e = row[jj];
            const int r0 = e.packed & 0xFFF, u = (e.packed >> 12) & 0xFFF, fl = e.packed >> 24;
            float f00 = 0.f, f01 = 0.f, f10 = 0.f, f11 = 0.f, g00 = 0.f, g01 = 0.f, g10 = 0.f, g11 = 0.f;
            if (fl & 1) { f00 = tile_at(mf, n, r0, u); g00 = tile_at(mg, n, r0, u); }
            if (fl & 2) { f01 = tile_at(mf, n, r0, u + 1); g01 = tile_at(mg, n, r0, u + 1); }
            if (fl & 4) { f10 = tile_at(mf, n, r0 + 1, u); g10 = tile_at(mg, n, r0 + 1, u); }
            if (fl & 8) { f11 = tile_at(mf, n, r0 + 1, u + 1); g11 = tile_at(mg, n, r0 + 1, u + 1); }
            af += (double)bilerp(e.fr, e.fc, f00, f01, f10, f11);
            ag += (double)bilerp(e.fr, e.fc, g00, g01, g10, g11);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            af += __shfl_xor_sync(0xffffffffu, af, o);
            ag += __shfl_xor_sync(0xffffffffu, ag, o);
        }
        if (lane == 0) {
            // wrap_pad (imageops.cpp:101-113): padded row q holds profile row (q - pad) mod nt
            for (int q = i + pad; q < L; q += nt) {
                A[q] = af;
                B[q] = ag;
            }
            for (int q = i + pad - nt; q >= 0; q -= nt) {
                A[q] = af;
                B[q] = ag;
            }
        }
    }
    __syncthreads();
    // s[k] = (1/C) sum_q A[q] B[(q + lag) mod L], lag = k - nt/2
    const double invC = 1.0 / (double)p.C;
    double best_v = -INFINITY;
    int best_i = 0x7fffffff;
    for (int k = threadIdx.x; k < nt; k += kPolarThreads) {
        const int lag = k - nt / 2;
        double acc = 0.0;
        if (lag >= 0) {
            for (int q = 0; q < L - lag; ++q) acc = fma(A[q], B[q + lag], acc);
            for (int q = L - lag; q < L; ++q) acc = fma(A[q], B[q + lag - L], acc);
        } else {
            for (int q = 0; q < -lag; ++q) acc = fma(A[q], B[q + lag + L], acc);
            for (int q = -lag; q < L; ++q) acc = fma(A[q], B[q + lag], acc);
        }
        const double sv = acc * invC;
        s[k] = sv;
        if (sv > best_v) {  // k increases per thread: strict > keeps the lowest index
            best_v = sv;
            best_i = k;
        }
    }
    // block argmax, ties -> lowest index (matcher.cpp:47-53)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best_v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (ov > best_v || (ov == best_v && oi < best_i)) {
            best_v = ov;
            best_i = oi;
        }
    }
    if (lane == 0) {
        red_v[warp] = best_v;
        red_i[warp] = best_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nwarps; ++w)
            if (red_v[w] > best_v || (red_v[w] == best_v && red_i[w] < best_i)) {
                best_v = red_v[w];
                best_i = red_i[w];
            }
        // soft_argmax over the n_theta x 1 surface (matcher.cpp:57-93)
        const int pk = best_i;
        const int r0 = max(0, pk - p.window), r1 = min(nt - 1, pk + p.window);
        double scale = 1.0;
        if (p.normalize) {
            double m = 0.0;
            for (int r = r0; r <= r1; ++r) m = fmax(m, fabs(s[r]));
            if (m > 0.0) scale = 1.0 / m;
        }
        const double top = s[pk] * scale;
        double wsum = 0.0, rsum = 0.0;
        for (int r = r0; r <= r1; ++r) {
            const double w = exp(p.t_theta * (s[r] * scale - top));
            wsum += w;
            rsum += w * ((r - nt / 2) * p.delta_theta);
        }
        const double theta = rsum / wsum;
        rs->theta = theta;
        double sn, cs;
        sincos(-theta, &sn, &cs);
        rs->st = sn;
        rs->ct = cs;
        rs->identity = (-theta == 0.0);
        rs->peak = s[pk];
        rs->hard = (pk - nt / 2) * p.delta_theta;
        rs->bin = pk;
        if (p.theta_only) p.theta_only[pair] = theta;
    }
    if (p.theta_surf) {
        __syncthreads();
        for (int k = threadIdx.x; k < nt; k += kPolarThreads) p.theta_surf[(size_t)pair * nt + k] = s[k];
    }
}

__global__ void k_theta_in(Params p) {
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= p.batch) return;
    const double theta = p.theta_in[pair];
    RotState* rs = p.rot + pair;
    rs->theta = theta;
    double sn, cs;
    sincos(-theta, &sn, &cs);
    rs->st = sn;
    rs->ct = cs;
    rs->identity = (-theta == 0.0);
    rs->peak = 0.0;
    rs->hard = 0.0;
    rs->bin = 0;
}

// ---------------------------------------------------------------- K3
// Row y of the translation stage: f~ row and the de-rotated g~ row
// (rotate_bilinear(g~, -theta), imageops.cpp:61-79, exact fp64 index map),
// packed z = f~ + i g~r; the 2N-point row transform of the zero-padded row
// is E = FFT_N(z) (even bins) and O = FFT_N(z W_2N^x) (odd bins); then the
// real spectra F = (Z[k] + conj Z[2N-k]) / 2, G = (Z[k] - conj Z[2N-k]) / 2i,
// k in [0, N], written transposed as fgt[k][y].
template <int N>
__global__ void __launch_bounds__(kRowThreads) k_xlat_rows(Params p) {
    constexpr int T = N / 16;
    constexpr int RPB = rows_per_block<N>();
    constexpr int KF = Cfg<N>::kFloats, KH = Cfg<N>::kHalf;
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    const int tr = threadIdx.x / T, t = threadIdx.x % T;
    const int y = blockIdx.x * RPB + tr;
    float* sa = smem + (2 * tr) * KF;
    float* sbb = smem + (2 * tr + 1) * KF;
    const RotState rs = p.rot[pair];
    const float* ft = p.ft + (size_t)pair * N * N;
    const float* gt = p.gt + (size_t)pair * N * N;
    const double c0 = (N - 1) / 2.0;
    const double vv = y - c0;
    float2 v[16], w[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int x = t + m * T;
        const float fv = ft[(size_t)y * N + x];
        float gv;
        if (rs.identity) {
            gv = gt[(size_t)y * N + x];
        } else {
            const double u = x - c0;
            // (c + st*u) + ct*v and (c + ct*u) - st*v, no contraction
            const double sr = __dadd_rn(__dadd_rn(c0, __dmul_rn(rs.st, u)), __dmul_rn(rs.ct, vv));
            const double sc = __dsub_rn(__dadd_rn(c0, __dmul_rn(rs.ct, u)), __dmul_rn(rs.st, vv));
            const double r0f = floor(sr), c0f = floor(sc);
            const int r0 = (int)r0f, cc0 = (int)c0f;
            const float fr = (float)(sr - r0f), fc = (float)(sc - c0f);
            const bool rin0 = (unsigned)r0 < (unsigned)N, rin1 = (unsigned)(r0 + 1) < (unsigned)N;
            const bool cin0 = (unsigned)cc0 < (unsigned)N, cin1 = (unsigned)(cc0 + 1) < (unsigned)N;
            const float a00 = (rin0 && cin0) ? gt[(size_t)r0 * N + cc0] : 0.0f;
            const float a01 = (rin0 && cin1) ? gt[(size_t)r0 * N + cc0 + 1] : 0.0f;
            const float a10 = (rin1 && cin0) ? gt[(size_t)(r0 + 1) * N + cc0] : 0.0f;
            const float a11 = (rin1 && cin1) ? gt[(size_t)(r0 + 1) * N + cc0 + 1] : 0.0f;
            gv = bilerp(fr, fc, a00, a01, a10, a11);
        }
        v[m] = make_float2(fv, gv);
        w[m] = cmul(v[m], __ldg(p.tw_2n + x));
    }
    fft_regs<N, -1>(v, t, sa, p.tw_n);
    fft_regs<N, -1>(w, t, sbb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int q = spad(t + m * T);
        sa[q] = v[m].x;
        sa[KH + q] = v[m].y;
        sbb[q] = w[m].x;
        sbb[KH + q] = w[m].y;
    }
    __syncthreads();
    // write fgt[k][y0 .. y0+RPB) with consecutive threads on consecutive y
    constexpr int KSTEP = kRowThreads / RPB;
    const int yl = threadIdx.x % RPB, kk = threadIdx.x / RPB;
    const int yy = blockIdx.x * RPB + yl;
    const float* ea = smem + (2 * yl) * KF;      // E of row yy
    const float* ob = smem + (2 * yl + 1) * KF;  // O of row yy
    float4* dst = p.fgt + (size_t)pair * (N + 1) * N;
    for (int k = kk; k <= N; k += KSTEP) {
        // Z[k]: even k -> E[k/2], odd k -> O[(k-1)/2]; partner Z[2N-k]
        const int kp = (2 * N - k) & (2 * N - 1);
        float2 z1, z2;
        if (k & 1) {
            const int q = spad(k >> 1);
            z1 = make_float2(ob[q], ob[KH + q]);
        } else {
            const int q = spad(k >> 1);
            z1 = make_float2(ea[q], ea[KH + q]);
        }
        if (kp & 1) {
            const int q = spad(kp >> 1);
            z2 = make_float2(ob[q], ob[KH + q]);
        } else {
            const int q = spad(kp >> 1);
            z2 = make_float2(ea[q], ea[KH + q]);
        }
        // F = (z1 + conj z2)/2 ; G = (z1 - conj z2)/(2i) = (im, -re)/2 of (z1 - conj z2)
        const float Fr = 0.5f * (z1.x + z2.x), Fi = 0.5f * (z1.y - z2.y);
        const float dr = z1.x - z2.x, di = z1.y + z2.y;
        const float Gr = 0.5f * di, Gi = -0.5f * dr;
        dst[(size_t)k * N + yy] = make_float4(Fr, Fi, Gr, Gi);
    }
}

// ---------------------------------------------------------------- K4
// Column k of the row spectra: 2N-point transforms of the half-zero columns
// F[:,k], G[:,k] (each as even/odd N-point FFTs), X = conj(F) G, inverse with
// output pruning to the N lags ky in [-N/2, N/2):
//   Y[ky] = e[j] + W_2N^{-j} o[j] (j < N/2, ky = j), e[j] - W_2N^{-j} o[j] (ky = j - N)
// with e = IFFT_N(X_even), o = IFFT_N(X_odd). Rows are stored by surface row
// i = half - ky (the world-flipped crop of matcher.cpp:171-182).
template <int N>
__global__ void __launch_bounds__(N / 2) k_xlat_cols(Params p) {
    constexpr int T = N / 16;
    constexpr int KF = Cfg<N>::kFloats;
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    const int c = threadIdx.x / T, t = threadIdx.x % T;
    const int k = blockIdx.x * 8 + c;
    const bool live = k <= N;  // last block holds only column N
    const int kk = live ? k : N;
    float* sb = smem + c * KF;
    const float4* src = p.fgt + ((size_t)pair * (N + 1) + kk) * N;
    // the [row][8 columns] output tile lives after the 8 FFT buffers
    float2* tile = reinterpret_cast<float2*>(smem + 8 * KF);
    constexpr int half = N / 2 - 1;
    float2 a[16], b[16];
    // odd bins first: tile <- +-W_2N^{-j} o[j]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const float4 q = src[t + m * T];
        const float2 tw = __ldg(p.tw_2n + t + m * T);
        a[m] = cmul(make_float2(q.x, q.y), tw);
        b[m] = cmul(make_float2(q.z, q.w), tw);
    }
    fft_regs<N, -1>(a, t, sb, p.tw_n);
    fft_regs<N, -1>(b, t, sb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) a[m] = cmul(cconj(a[m]), b[m]);
    fft_regs<N, +1>(a, t, sb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int j = t + m * T;
        const float2 wo = cmul(cconj(__ldg(p.tw_2n + j)), a[m]);  // W_2N^{-j} o[j]
        const int ky = j < N / 2 ? j : j - N;
        tile[(half - ky) * 8 + c] = j < N / 2 ? wo : make_float2(-wo.x, -wo.y);
    }
    // even bins: tile += e[j] (same thread, same slot: no barrier needed)
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const float4 q = src[t + m * T];
        a[m] = make_float2(q.x, q.y);
        b[m] = make_float2(q.z, q.w);
    }
    fft_regs<N, -1>(a, t, sb, p.tw_n);
    fft_regs<N, -1>(b, t, sb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) a[m] = cmul(cconj(a[m]), b[m]);
    fft_regs<N, +1>(a, t, sb, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int j = t + m * T;
        const int ky = j < N / 2 ? j : j - N;
        float2* slot = tile + (half - ky) * 8 + c;
        *slot = cadd(*slot, a[m]);
    }
    __syncthreads();
    float2* dst = p.zbuf + (size_t)pair * N * (N + 1);
    const int ncols = min(8, N + 1 - blockIdx.x * 8);
    for (int o = threadIdx.x; o < N * 8; o += N / 2) {
        const int i = o >> 3, cc = o & 7;
        if (cc < ncols) dst[(size_t)i * (N + 1) + blockIdx.x * 8 + cc] = tile[o];
    }
}

// ---------------------------------------------------------------- K5
// Surface row i: the length-2N real inverse along x of the Hermitian half
// Y[0..N] as one N-point complex inverse FFT:
//   A[k] = Y[k] + conj Y[N-k], B[k] = (Y[k] - conj Y[N-k]) W_2N^{-k},
//   z = IFFT_N(A + iB), x[2n] = Re z[n], x[2n+1] = Im z[n];
// scaled by 1/P^2 (spectral.cpp:145), cropped to lags [-(N/2-1), N/2]
// (surface col j = lag + half), plus this block's hard argmax.
template <int N>
__global__ void __launch_bounds__(kRowThreads) k_xlat_out(Params p) {
    constexpr int T = N / 16;
    constexpr int RPB = rows_per_block<N>();
    extern __shared__ float smem[];
    __shared__ float red_v[kRowThreads / 32];
    __shared__ int red_i[kRowThreads / 32];
    const int pair = blockIdx.y;
    const int tr = threadIdx.x / T, t = threadIdx.x % T;
    const int i = blockIdx.x * RPB + tr;
    float* sb = smem + tr * Cfg<N>::kFloats;
    const float2* yrow = p.zbuf + ((size_t)pair * N + i) * (N + 1);
    float2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int k = t + m * T;
        const float2 a = yrow[k], b = cconj(yrow[N - k]);
        const float2 A = cadd(a, b);
        const float2 B = cmul(csub(a, b), cconj(__ldg(p.tw_2n + k)));
        v[m] = make_float2(A.x - B.y, A.y + B.x);  // A + iB
    }
    fft_regs<N, +1>(v, t, sb, p.tw_n);
    const float scale = 1.0f / ((float)(2 * N) * (float)(2 * N));
    constexpr int half = N / 2 - 1;
    float* srow = (p.xy_surf ? p.xy_surf : p.surf) + ((size_t)pair * N + i) * N;
    float best_v = -INFINITY;
    int best_i = 0x7fffffff;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int nn = t + m * T;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int pos = 2 * nn + h;                       // position in [0, 2N)
            const int lag = pos <= N / 2 ? pos : pos - 2 * N;  // valid when in [-(N/2-1), N/2]
            if (lag >= -half && lag <= N / 2) {
                const float val = (h ? v[m].y : v[m].x) * scale;
                const int j = lag + half;
                srow[j] = val;
                const int li = i * N + j;
                if (val > best_v || (val == best_v && li < best_i)) {
                    best_v = val;
                    best_i = li;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best_v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (ov > best_v || (ov == best_v && oi < best_i)) {
            best_v = ov;
            best_i = oi;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red_v[warp] = best_v;
        red_i[warp] = best_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kRowThreads / 32; ++w)
            if (red_v[w] > best_v || (red_v[w] == best_v && red_i[w] < best_i)) {
                best_v = red_v[w];
                best_i = red_i[w];
            }
        p.part[(size_t)pair * gridDim.x + blockIdx.x] = Partial{best_v, best_i};
    }
}

// ---------------------------------------------------------------- K6
constexpr int kFinThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < kFinThreads / 32; ++w) r += sh[w];
    return r;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = sh[0];
    for (int w = 1; w < kFinThreads / 32; ++w) r = fmax(r, sh[w]);
    return r;
}

__global__ void __launch_bounds__(kFinThreads) k_finalize(Params p, int nparts) {
    __shared__ double sh[kFinThreads / 32];
    __shared__ float pk_v;
    __shared__ int pk_i;
    const int pair = blockIdx.x;
    const int n = p.n;
    if (threadIdx.x == 0) {
        const Partial* pp = p.part + (size_t)pair * nparts;
        float bv = pp[0].val;
        int bi = pp[0].idx;
        for (int b = 1; b < nparts; ++b)
            if (pp[b].val > bv || (pp[b].val == bv && pp[b].idx < bi)) {
                bv = pp[b].val;
                bi = pp[b].idx;
            }
        pk_v = bv;
        pk_i = bi;
    }
    __syncthreads();
    const float* surf = (p.xy_surf ? p.xy_surf : p.surf) + (size_t)pair * n * n;
    const int pr = pk_i / n, pc = pk_i % n;
    const int w = p.window;
    const int r0 = max(0, pr - w), r1 = min(n - 1, pr + w);
    const int c0 = max(0, pc - w), c1 = min(n - 1, pc + w);
    const int wr = r1 - r0 + 1, wc = c1 - c0 + 1;
    double scale = 1.0;
    if (p.normalize) {
        double m = 0.0;
        for (int q = threadIdx.x; q < wr * wc; q += kFinThreads)
            m = fmax(m, fabs((double)surf[(size_t)(r0 + q / wc) * n + c0 + q % wc]));
        m = block_max(m, sh);
        if (m > 0.0) scale = 1.0 / m;
    }
    const double top = (double)pk_v * scale;
    const int half = (n - 1) / 2;
    double ws = 0.0, rsum = 0.0, csum = 0.0;
    for (int q = threadIdx.x; q < wr * wc; q += kFinThreads) {
        const int r = r0 + q / wc, cc = c0 + q % wc;
        const double wgt = exp(p.t_xy * ((double)surf[(size_t)r * n + cc] * scale - top));
        ws += wgt;
        rsum += wgt * ((r - half) * p.delta);
        csum += wgt * ((cc - half) * p.delta);
    }
    ws = block_sum(ws, sh);
    rsum = block_sum(rsum, sh);
    csum = block_sum(csum, sh);
    if (threadIdx.x == 0) {
        const RotState rs = p.rot[pair];
        const double ty_ = rsum / ws, tx_ = csum / ws;
        double sn, cs;
        sincos(rs.theta, &sn, &cs);  // rotate_vec (geometry.cpp:31-35)
        const double tx = cs * tx_ - sn * ty_;
        const double ty = sn * tx_ + cs * ty_;
        if (p.txy_only) {
            p.txy_only[2 * pair] = tx;
            p.txy_only[2 * pair + 1] = ty;
        }
        if (p.out) {
            const double two_pi = 6.283185307179586;
            const double pi = 3.141592653589793;
            double th = fmod(rs.theta, two_pi);  // normalize_angle (geometry.cpp:9-14)
            if (th <= -pi) th += two_pi;
            if (th > pi) th -= two_pi;
            fscan_pair_result o;
            o.theta = th;
            o.tx = tx;
            o.ty = ty;
            o.theta_hard = rs.hard;
            o.theta_peak = rs.peak;
            o.xy_hard_x = (pc - half) * p.delta;
            o.xy_hard_y = (pr - half) * p.delta;
            o.xy_peak = (double)pk_v;
            o.theta_bin = rs.bin;
            o.xy_row = pr;
            o.xy_col = pc;
            const int fl = p.flags[pair];
            o.status = (fl & 2) ? FSCAN_ERR_MASK_RANGE : ((fl & 1) ? FSCAN_ERR_NONFINITE : FSCAN_OK);
            p.out[pair] = o;
        }
    }
}

// band magnitude stage output: tiled [2][N/16][N][8] (f only) -> [N][N/2]
__global__ void k_mag_unpack(Params p) {
    const int n = p.n;
    const int pair = blockIdx.y;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)n * (n / 2)) return;
    const int vc = (int)(idx / (n / 2)), u = (int)(idx % (n / 2));
    const float* m = p.mag + (size_t)pair * 2 * n * (n / 2);
    p.mag_out[(size_t)pair * n * (n / 2) + idx] = m[((size_t)(u >> 3) * n + vc) * 8 + (u & 7)];
}

__global__ void k_polar_to_cart(const float* polar, int n_az, int n_range, double res, int n,
                                double delta, float* out) {
    const int pair = blockIdx.y;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)n * n) return;
    const int r = (int)(idx / n), c = (int)(idx % n);
    out[(size_t)pair * n * n + idx] = (float)fscan_k0::polar_cell(
        polar + (size_t)pair * n_az * n_range, n_az, n_range, res, n, delta, r, c);
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return cudaSuccess;
}

#define FSCAN_DISPATCH_N(n, FN)                   \
    switch (n) {                                  \
        case 64: return FN<64>(p, s);             \
        case 128: return FN<128>(p, s);           \
        case 256: return FN<256>(p, s);           \
        case 512: return FN<512>(p, s);           \
        case 1024: return FN<1024>(p, s);         \
        default: return cudaErrorInvalidValue;    \
    }

template <int N>
cudaError_t rot_rows(const Params& p, cudaStream_t s) {
    constexpr int RPB = rows_per_block<N>();
    const size_t sm = (size_t)RPB * Cfg<N>::kFloats * sizeof(float);
    cudaError_t e = set_smem(k_rot_rows<N>, sm);
    if (e != cudaSuccess) return e;
    k_rot_rows<N><<<dim3(N / RPB, p.batch), kRowThreads, sm, s>>>(p);
    return cudaGetLastError();
}

template <int N>
cudaError_t rot_cols(const Params& p, cudaStream_t s) {
    const size_t sm = (size_t)16 * Cfg<N>::kFloats * sizeof(float);
    cudaError_t e = set_smem(k_rot_cols<N>, sm);
    if (e != cudaSuccess) return e;
    k_rot_cols<N><<<dim3(N / 16, p.batch), N, sm, s>>>(p);
    return cudaGetLastError();
}

template <int N>
cudaError_t xlat_rows(const Params& p, cudaStream_t s) {
    constexpr int RPB = rows_per_block<N>();
    const size_t sm = (size_t)2 * RPB * Cfg<N>::kFloats * sizeof(float);
    cudaError_t e = set_smem(k_xlat_rows<N>, sm);
    if (e != cudaSuccess) return e;
    k_xlat_rows<N><<<dim3(N / RPB, p.batch), kRowThreads, sm, s>>>(p);
    return cudaGetLastError();
}

template <int N>
cudaError_t xlat_cols(const Params& p, cudaStream_t s) {
    const size_t sm = (size_t)8 * Cfg<N>::kFloats * sizeof(float) + (size_t)8 * N * sizeof(float2);
    cudaError_t e = set_smem(k_xlat_cols<N>, sm);
    if (e != cudaSuccess) return e;
    k_xlat_cols<N><<<dim3((N + 1 + 7) / 8, p.batch), N / 2, sm, s>>>(p);
    return cudaGetLastError();
}

template <int N>
cudaError_t xlat_out(const Params& p, cudaStream_t s) {
    constexpr int RPB = rows_per_block<N>();
    const size_t sm = (size_t)RPB * Cfg<N>::kFloats * sizeof(float);
    cudaError_t e = set_smem(k_xlat_out<N>, sm);
    if (e != cudaSuccess) return e;
    k_xlat_out<N><<<dim3(N / RPB, p.batch), kRowThreads, sm, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

int rows_per_block_out(int n) {
    switch (n) {
        case 64: return rows_per_block<64>();
        case 128: return rows_per_block<128>();
        case 256: return rows_per_block<256>();
        case 512: return rows_per_block<512>();
        case 1024: return rows_per_block<1024>();
        default: return 1;
    }
}

cudaError_t launch_rot_rows(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, rot_rows) }
cudaError_t launch_rot_cols(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, rot_cols) }
cudaError_t launch_xlat_rows(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, xlat_rows) }
cudaError_t launch_xlat_cols(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, xlat_cols) }
cudaError_t launch_xlat_out(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, xlat_out) }

cudaError_t launch_rot_polar(const Params& p, cudaStream_t s) {
    const size_t sm = (size_t)(2 * p.L + p.n_theta + 32) * sizeof(double) + 32 * sizeof(int);
    cudaError_t e = set_smem(k_rot_polar, sm);
    if (e != cudaSuccess) return e;
    k_rot_polar<<<p.batch, kPolarThreads, sm, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_theta_in(const Params& p, cudaStream_t s) {
    k_theta_in<<<(p.batch + 127) / 128, 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Params& p, cudaStream_t s) {
    k_finalize<<<p.batch, kFinThreads, 0, s>>>(p, p.n / rows_per_block_out(p.n));
    return cudaGetLastError();
}

cudaError_t launch_mag_unpack(const Params& p, cudaStream_t s) {
    const size_t total = (size_t)p.n * (p.n / 2);
    k_mag_unpack<<<dim3((unsigned)((total + 255) / 256), p.batch), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_polar_to_cart(const float* d_polar, int batch, int n_az, int n_range, double range_res,
                                 int n, double delta, float* d_out, cudaStream_t stream) {
    const size_t total = (size_t)n * n;
    k_polar_to_cart<<<dim3((unsigned)((total + 255) / 256), batch), 256, 0, stream>>>(
        d_polar, n_az, n_range, range_res, n, delta, d_out);
    return cudaGetLastError();
}

}  // namespace fscan_detail
