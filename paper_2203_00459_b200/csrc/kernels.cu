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

#include <algorithm>
#include <math.h>
#include <stdlib.h>
#include <stdint.h>

#include "fft.cuh"
#include "pipeline.h"
#include "polar.h"


#ifndef FSCAN_K5_TWO_PASS
#define FSCAN_K5_TWO_PASS 1  // K5 block maxima only + soft-argmax window rows recomputed (k_xlat_out modes)
#endif
#ifndef FSCAN_K5_TWO_PASS_MIN_N
#define FSCAN_K5_TWO_PASS_MIN_N 512
#endif
// Packed complex add / subtract (FADD2, fft.cuh) in the FFT butterflies of grid
// sides >= 512: C4 / C5 / C3 +1.2% each; at N = 256 the 64-pair batch (C2) ran
// 1.5% slower with it, so the smaller grids keep the scalar adds.
#ifndef FSCAN_F32X2_MIN_N
#define FSCAN_F32X2_MIN_N 512
#endif
#ifndef FSCAN_PK_K3
#define FSCAN_PK_K3 1
#endif
#ifndef FSCAN_PK_K4
#define FSCAN_PK_K4 1
#endif
#ifndef FSCAN_PK_K5
#define FSCAN_PK_K5 1
#endif
template <int N>
constexpr bool kPk = fscan_fft::kF32x2Add && N >= FSCAN_F32X2_MIN_N;  // K4, K5
// K3 only at N = 512 (6.48 -> 6.33 ms; at N = 1024 7.34 -> 7.62 ms); the
// rotation-stage transforms (K1a DRAM-bound, K1b 2.54 -> 2.62 ms at N = 1024)
// keep the scalar adds
template <int N>
constexpr bool kPkRows = kPk<N> && N < 1024;
#ifndef FSCAN_K3_U
#define FSCAN_K3_U 4  // K3 gather: cells per thread with their loads in flight together
#endif

namespace fscan_detail {

using fscan_fft::cadd;
using fscan_fft::cconj;
using fscan_fft::cmul;
using fscan_fft::csub;
using fscan_fft::fft_regs;
using fscan_fft::Geom;
using fscan_fft::Lay;
using fscan_fft::part_floats;

namespace {

// one-shot mbarrier + TMA bulk copy global -> shared (cp.async.bulk)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Programmatic dependent launch (griddepcontrol, sm_90+): the pipeline kernels
// of a chunk are launched with programmatic stream serialisation when the
// context asks for it (Params::pdl), so a kernel's CTAs are scheduled while its
// predecessor on the stream drains instead of after it has completed and the
// launch has gone through the front end. pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible: every read of data
// another kernel produced, and every global write, comes after it (only kernel
// parameters and the context's constant tables are read before). pdl_trigger()
// lets this grid's own dependent launch once every CTA of this grid runs
// (after pdl_wait, so at most one grid per stream is waiting). Both are no-ops
// for a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

#ifdef FSCAN_K3_FT_LDG
constexpr bool kK3FtTma = false;  // A/B: K3 loads f~ per thread from global
#else
constexpr bool kK3FtTma = true;
#endif

// K1a CTA size: 128 threads (4 rows at N = 512) leave room for K1a CTAs next
// to the compute-bound translation kernels of the other lane (measured -5% K1a)
#ifndef FSCAN_K1A_THREADS
#define FSCAN_K1A_THREADS 128
#endif
constexpr int kRowThreads = FSCAN_K1A_THREADS;
// K1a residency: at N = 512, 7 CTAs of 128 threads per SM (<= 72 registers);
// without a bound ptxas takes 80 with the padded layout (and 132 with an
// explicit minBlocks of 1)
template <int N>
__host__ __device__ constexpr int k1a_minb() {
    return N >= 1024 ? 6 : (N == 512 ? 7 : 8);
}
#ifdef FSCAN_K1A_MINB
#define FSCAN_K1A_BOUNDS __launch_bounds__(kRowThreads, FSCAN_K1A_MINB)
#else
#define FSCAN_K1A_BOUNDS __launch_bounds__(kRowThreads, k1a_minb<N>())
#endif

template <int N>
using RowG = Geom<N, kRowThreads>;

template <int N>
__host__ __device__ constexpr int rows_per_block() {
    return RowG<N>::PER_CTA;
}

__device__ __forceinline__ float bilerp(float fr, float fc, float a00, float a01, float a10, float a11) {
    // sample_bilinear (imageops.cpp:24-25) operation order, fp32
    return (1.0f - fr) * ((1.0f - fc) * a00 + fc * a01) + fr * ((1.0f - fc) * a10 + fc * a11);
}

// (|F|,|G|) columns per magnitude tile row (4 measured equal: faster K2a
// gather, slower K1b stores)
constexpr int kTileW = 8;
__device__ __forceinline__ const float2* tile_at(const float2* m, int n, int r, int u) {
    return m + ((size_t)(u / kTileW) * n + r) * kTileW + (u % kTileW);
}

// K1a -> K1b spectrum columns in K1b's column blocks: per pair, NB = zcols / U
// direct blocks (columns b U + c) then NB mirror blocks (columns (N - b U - c)
// mod N), each [N rows][U] float2 — exactly the 2U columns one K1b CTA
// transforms, contiguous, so the CTA fetches them with two bulk copies instead
// of 16 scattered 64-byte row pieces per thread (U = k1b_u<N>())
// FOLD1 fold twiddles from one table read per thread times W_8 / W_3 constants
// instead of two table reads per site (C5 +0.3%)
#ifdef FSCAN_K4_FOLD1_TABLE
constexpr bool kK4Fold1Base = false;  // A/B
#else
constexpr bool kK4Fold1Base = true;
#endif
#ifdef FSCAN_K1A_FLAG_CMP
constexpr bool kK1aFlagAcc = false;  // A/B: per-element compares for the input flags
#else
constexpr bool kK1aFlagAcc = true;
#endif
#ifndef FSCAN_K1B_U512
#define FSCAN_K1B_U512 8  // K1b output columns per CTA at N = 512
#endif
#ifdef FSCAN_K1B_ROWMAJOR
constexpr bool kK1bBlocks = false;  // A/B: row-major spectrum, per-thread column loads (rounds 1-2)
#else
constexpr bool kK1bBlocks = true;
#endif
template <int N>
__host__ __device__ constexpr int k1b_u() {
    return N >= 1024 ? 4 : (N == 512 ? FSCAN_K1B_U512 : 8);
}
// float2 offset of column slot c of direct (mirror = 0) or mirror (1) block b, row y
template <int N>
__device__ __forceinline__ size_t k1b_at(int pair, int zcols, int mirror, int w, int y) {
    constexpr int U = k1b_u<N>();
    const int blk = mirror * (zcols / U) + w / U;
    return (size_t)pair * N * N + ((size_t)blk * N + y) * U + (w % U);
}

// ---------------------------------------------------------------- K1a
// rows of f~ = f*mf and g~ = g*mg: write the masked scans (translation stage
// input), window by the separable Hann w[r]*w[c], FFT the packed row
// z = f~w + i g~w.
// the scans and masks are read once per call: A/B (FSCAN_K1A_STREAM) loads them
// with the evict-first hint (ld.global.cs) so they do not displace the other
// lanes' intermediates in L2
#if defined(FSCAN_K1A_STREAM) && FSCAN_K1A_STREAM == 2
// the read-only path as __ldg, the L2 line marked evict-first by a cache policy
__device__ __forceinline__ float ld_in(const float* p) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
#elif defined(FSCAN_K1A_STREAM)
__device__ __forceinline__ float ld_in(const float* p) { return __ldcs(p); }  // measured: K1a 4.95 -> 8.4 ms
#else
__device__ __forceinline__ float ld_in(const float* p) { return __ldg(p); }
#endif
template <int N>
__global__ void FSCAN_K1A_BOUNDS k_rot_rows(Params p) {
    pdl_enter();
    using G = RowG<N>;
    constexpr int T = G::T;
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    int tr, t;
    G::map(threadIdx.x, tr, t);
    const int y = blockIdx.x * G::PER_CTA + tr;
    const auto lay = G::lay(smem, tr);
    const size_t base = ((size_t)pair * N + y) * N;
    // the two real grids packed into this transform: scans `pair` of f and g, or
    // in chain mode (odometry) scans 2*pair and 2*pair+1 of one sequence (the
    // last one duplicated for an odd count), masked copies written per scan
    const float *fp, *gp, *mfp = nullptr, *mgp = nullptr;
    float *ftp, *gtp;
    const size_t row = (size_t)y * N;
    if (p.chain) {
        const size_t fi = 2 * (size_t)pair, gi = (size_t)min(2 * pair + 1, p.n_scans - 1);
        fp = p.f + fi * N * N + row;
        gp = p.f + gi * N * N + row;
        if (p.mf) {
            mfp = p.mf + fi * N * N + row;
            mgp = p.mf + gi * N * N + row;
        }
        ftp = p.ft + fi * N * N + row;
        gtp = p.ft + gi * N * N + row;
    } else {
        fp = p.f + base;
        gp = p.g + base;
        if (p.mf) {
            mfp = p.mf + base;
            mgp = p.mg + base;
        }
        ftp = p.ft + base;
        gtp = p.gt + base;
    }
    const float hy = p.hann[y];
    int badf = 0, badg = 0;  // bit0 non-finite, bit1 mask outside [0, 1]
    float2 v[16];
    auto finish = [&](int m, int x, float fv, float gv) {
        ftp[x] = fv;
        gtp[x] = gv;
        const float w = hy * __ldg(p.hann + x);
        v[m] = make_float2(fv * w, gv * w);
    };
    if constexpr (kK1aFlagAcc) {
        // flags as running values instead of per-element compares: fma(x, 0, c)
        // turns NaN for any non-finite x (inf * 0 = NaN) and stays 0 otherwise;
        // the masks' range as a running min / max (fminf / fmaxf skip NaN, which
        // the fma check then catches) — the same tests as !isfinite(f * m) and
        // !(m >= 0 && m <= 1), per scan
        float cf = 0.f, cg = 0.f, ca = 0.f, cb = 0.f, alo = 0.f, ahi = 1.f, blo = 0.f, bhi = 1.f;
        if (mfp) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int x = t + m * T;
                const float a = ld_in(mfp + x), b = ld_in(mgp + x);
                const float fv = ld_in(fp + x) * a, gv = ld_in(gp + x) * b;
                alo = fminf(alo, a), ahi = fmaxf(ahi, a), blo = fminf(blo, b), bhi = fmaxf(bhi, b);
                ca = fmaf(a, 0.f, ca), cb = fmaf(b, 0.f, cb);
                cf = fmaf(fv, 0.f, cf), cg = fmaf(gv, 0.f, cg);
                finish(m, x, fv, gv);
            }
        } else {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int x = t + m * T;
                const float fv = __ldg(fp + x), gv = __ldg(gp + x);
                cf = fmaf(fv, 0.f, cf), cg = fmaf(gv, 0.f, cg);
                finish(m, x, fv, gv);
            }
        }
        badf = (cf != cf ? 1 : 0) | ((alo < 0.f || ahi > 1.f || ca != ca) ? 2 : 0);
        badg = (cg != cg ? 1 : 0) | ((blo < 0.f || bhi > 1.f || cb != cb) ? 2 : 0);
    } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int x = t + m * T;
            float fv = __ldg(fp + x);
            float gv = __ldg(gp + x);
            if (mfp) {
                const float a = __ldg(mfp + x), b = __ldg(mgp + x);
                if (!(a >= 0.0f && a <= 1.0f)) badf |= 2;
                if (!(b >= 0.0f && b <= 1.0f)) badg |= 2;
                fv *= a;
                gv *= b;
            }
            if (!isfinite(fv)) badf |= 1;
            if (!isfinite(gv)) badg |= 1;
            finish(m, x, fv, gv);
        }
    }
    fft_regs<N, -1, (G::T <= 32), false>(v, t, lay, p.tw_n);  // a row per warp (or two warps at N = 1024)
    constexpr int UB = k1b_u<N>();
    // HOIST: with U dividing T, column x = t + m T sits in direct block t / U + m T / U
    // and its mirror N - x in mirror block (N - t) / U - m T / U, both at a fixed
    // slot: one base address each, compile-time offsets (x = 0's mirror, column
    // 0 itself, is stored separately)
    constexpr bool HOIST = kK1bBlocks && T % UB == 0;
    [[maybe_unused]] float2* zd = p.zbuf + k1b_at<N>(pair, p.zcols, 0, t, y);
    [[maybe_unused]] float2* zm = p.zbuf + k1b_at<N>(pair, p.zcols, 1, N - t, y);  // (t = 0: one block past, m >= 1 only)
    if constexpr (HOIST)
        if (t == 0) p.zbuf[k1b_at<N>(pair, p.zcols, 1, 0, y)] = v[0];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int x = t + m * T;
        if constexpr (HOIST) {
            constexpr int STEP = (T / UB) * N * UB;
            if (x < p.zcols) zd[m * STEP] = v[m];
            if (x > N - p.zcols) zm[-m * STEP] = v[m];
        } else if constexpr (kK1bBlocks) {
            // the columns K1b reads, in its column blocks (k1b_at)
            if (x < p.zcols) p.zbuf[k1b_at<N>(pair, p.zcols, 0, x, y)] = v[m];
            if (x == 0 || x > N - p.zcols) p.zbuf[k1b_at<N>(pair, p.zcols, 1, (N - x) & (N - 1), y)] = v[m];
        } else if (x < p.zcols || x > N - p.zcols) {
            p.zbuf[base + x] = v[m];  // columns K1b reads
        }
    }
    if (p.chain) {  // flags per scan of the sequence
        if (badf) atomicOr(p.flags + 2 * pair, badf);
        if (badg) atomicOr(p.flags + min(2 * pair + 1, p.n_scans - 1), badg);
    } else if (badf | badg) {
        atomicOr(p.flags + pair, badf | badg);
    }
}

// ---------------------------------------------------------------- K1b
// k1b_u<N>() output columns u in [u0, u0 + U) plus their mirrors (N-u) mod N,
// 2U interleaved column FFTs (column index fastest in the warp);
// F = (Z[v,u] + conj Z[-v,-u]) / 2, G = (Z[v,u] - conj Z[-v,-u]) / 2i;
// |F|, |G| times the annular band, written into the [N centred rows][8] tiles
// of (|F|, |G|) pairs (a CTA fills U of a tile's 8 columns).
// (N = 1024 at 4 columns: 512 threads instead of 1024; C5 +0.4%; N = 512 at
// 4 columns measured 0.8% slower than 8)
template <int N>
__host__ __device__ constexpr size_t k1b_smem_floats() {
    // exchange buffer, or (kK1bBlocks) the two staged blocks with the mirror block
    // 8 float2 further on (its half-warp reads then miss the direct block's banks)
    constexpr size_t ex = (size_t)part_floats<N, 2 * k1b_u<N>()>();
    constexpr size_t st = (size_t)2 * (2 * (size_t)N * k1b_u<N>() + 8);
    return kK1bBlocks && st > ex ? st : ex;
}

template <int N>
__global__ void __launch_bounds__(N / 16 * 2 * k1b_u<N>()) k_rot_cols(Params p) {
    pdl_enter();
    constexpr int U = k1b_u<N>(), CW = 2 * U;  // CW interleaved transforms per CTA
    constexpr int T = N / 16;
    constexpr int THREADS = T * CW;
    extern __shared__ float smem[];
    const int pair = blockIdx.y;
    const int u0 = blockIdx.x * U;
    const int c = threadIdx.x % CW, t = threadIdx.x / CW;
    [[maybe_unused]] const int col = c < U ? (u0 + c) : ((N - (u0 + c - U)) & (N - 1));
    float2* sbuf = reinterpret_cast<float2*>(smem);
    const Lay<CW> lay{sbuf, c};
    float2 v[16];
    if constexpr (kK1bBlocks) {
        // the CTA's direct and mirror column blocks by two bulk copies into the
        // exchange buffer's bytes (read into registers before the first exchange)
        constexpr unsigned BYTES = (unsigned)(N * U * sizeof(float2));
        constexpr int BOFF = N * U + 8;
        __shared__ uint64_t bar;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 2);
            bulk_load(sbuf, p.zbuf + k1b_at<N>(pair, p.zcols, 0, u0, 0), BYTES, &bar);
            bulk_load(sbuf + BOFF, p.zbuf + k1b_at<N>(pair, p.zcols, 1, u0, 0), BYTES, &bar);
        }
        __syncthreads();  // publishes the barrier's initialisation
        mbar_wait(&bar, 0);
        const float2* sb = sbuf + (c < U ? c : BOFF + c - U);
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = sb[(t + m * T) * U];
        __syncthreads();  // every staged value read before the exchange reuses the bytes
    } else {
        const float2* z = p.zbuf + (size_t)pair * N * N;
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = z[(size_t)(t + m * T) * N + col];
    }
    fft_regs<N, -1, false, false>(v, t, lay, p.tw_n);
#pragma unroll
    for (int m = 0; m < 16; ++m) lay.put(t + m * T, v[m]);
    __syncthreads();
    // (|F|, |G|) interleaved: one 8-byte load per tap in K2a
    float2* out = reinterpret_cast<float2*>(p.mag) + ((size_t)pair * (N / 16) + u0 / 8) * (size_t)(N * 8) + (u0 & 7);
#pragma unroll
    for (int q = 0; q < N * U / THREADS; ++q) {
        const int o = threadIdx.x + q * THREADS;  // o = v_c * U + cc
        const int cc = o % U, vc = o / U;
        const int vn = (vc + N / 2) & (N - 1);  // natural row of centred row vc
        const int vm = (N - vn) & (N - 1);      // row of -v
        const float2 z1 = Lay<CW>{sbuf, cc}.get(vn);
        const float2 z2 = Lay<CW>{sbuf, U + cc}.get(vm);
        const float fr = z1.x + z2.x, fi = z1.y - z2.y;  // Z1 + conj(Z2)
        const float gr = z1.x - z2.x, gi = z1.y + z2.y;  // Z1 - conj(Z2)
        const int2 bd = __ldg(p.band + vc);
        const int u = u0 + cc;
        const bool in = (u >= bd.x) && (u <= bd.y);
        const float2 mv = in ? make_float2(0.5f * fscan_fft::sqrt_fast(fr * fr + fi * fi), 0.5f * fscan_fft::sqrt_fast(gr * gr + gi * gi))
                             : make_float2(0.0f, 0.0f);
        out[vc * 8 + cc] = mv;  // tile [u0 / 8][v_c][u0 % 8 + cc]
    }
}

// ---------------------------------------------------------------- K2
constexpr int kPolarThreads = 512;
#ifndef FSCAN_K2B_SPLIT_BELOW
#define FSCAN_K2B_SPLIT_BELOW 64  // batches below this split K2b over several CTAs per pair
#endif

// K2b angular correlation: each thread owns kLags consecutive lags over one of
// polar_parts(nt) q-ranges, so that (lag blocks) x parts fills the CTA.
constexpr int kLags = 8;

__host__ __device__ inline int polar_parts(int nt) {
    const int blocks = (nt + kLags - 1) / kLags;
    const int np = kPolarThreads / (blocks > 0 ? blocks : 1);
    return np < 1 ? 1 : (np > 16 ? 16 : np);
}

// Bx is stored skewed by one double per 8 (lane stride kLags = 8 doubles maps
// to 9: conflict-free 64-bit shared loads)
__host__ __device__ inline int bx_skew(int j) { return j + (j >> 3); }
__host__ __device__ inline int bx_len(int L, int nt) { return bx_skew(L + nt + 2 * kLags) + 1; }


// K2a: radial sums of the bilinear polar resample (cart2pol) of |F| and |G|:
// one thread per azimuth row, walking its radii. The lanes of a warp are 32
// adjacent rays at the same radius, which sit within a few pixels of each
// other, so a warp-wide tap load touches few magnitude-tile lines (4 rows x 4
// (|F|,|G|) columns each) instead of the many a ray's consecutive radii span.
// fp64 sums per row, written to p.prof[pair][2][n_theta]; the tap table is
// radius-major ([n_live][n_theta]).
constexpr int kGatherThreads = 128;

// SPLIT (chain mode, odd pair k): |F| of scan k is the .y of transform k/2,
// |G| of scan k+1 the .x of transform k/2 + 1.
template <bool SPLIT>
__device__ __forceinline__ void gather_sums(const Params& p, const float2* m, int i, bool live, int rsub,
                                            double* prof) {
    const int nt = p.n_theta, n = p.n, n_live = p.n_live;
    const float2* m2 = m + p.mag_plane;  // the next transform's tiles (chain mode)
    const PolarTap* col = p.taps + (live ? i : 0);
    double af = 0.0, ag = 0.0;
    // a warp covers 8 azimuths x 4 radii per step (lane = 4 * azimuth + radius
    // phase): the 32 samples of one load instruction form a compact patch of the
    // magnitude plane instead of a 32-azimuth arc, so they touch fewer cache lines
    constexpr int U = 4;  // independent entries in flight per thread (memory-level parallelism)
    for (int j0 = rsub; j0 < n_live; j0 += 4 * U) {
        PolarTap e[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int j = j0 + 4 * q;
            e[q] = (live && j < n_live) ? col[(size_t)j * nt] : PolarTap{0, 0.f, 0.f, 0.f};  // flags 0: 0
        }
        float fv[U][4], gv[U][4];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int r0 = e[q].packed & 0xFFF, u = (e[q].packed >> 12) & 0xFFF, fl = e[q].packed >> 24;
#pragma unroll
            for (int tp = 0; tp < 4; ++tp) {
                const bool on = (fl >> tp) & 1;
                const int rr = r0 + (tp >> 1), uu = u + (tp & 1);
                if constexpr (SPLIT) {
                    fv[q][tp] = on ? __ldg(&tile_at(m, n, rr, uu)->y) : 0.f;
                    gv[q][tp] = on ? __ldg(&tile_at(m2, n, rr, uu)->x) : 0.f;
                } else {
                    const float2 v = on ? __ldg(tile_at(m, n, rr, uu)) : make_float2(0.f, 0.f);
                    fv[q][tp] = v.x;
                    gv[q][tp] = v.y;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            af += (double)bilerp(e[q].fr, e[q].fc, fv[q][0], fv[q][1], fv[q][2], fv[q][3]);
            ag += (double)bilerp(e[q].fr, e[q].fc, gv[q][0], gv[q][1], gv[q][2], gv[q][3]);
        }
    }
    // the four radius phases of an azimuth, summed in a fixed order
    af += __shfl_xor_sync(0xffffffffu, af, 1);
    ag += __shfl_xor_sync(0xffffffffu, ag, 1);
    af += __shfl_xor_sync(0xffffffffu, af, 2);
    ag += __shfl_xor_sync(0xffffffffu, ag, 2);
    if (live && rsub == 0) {
        prof[i] = af;
        prof[nt + i] = ag;
    }
}

// PB pairs per CTA (independent pairs only): every tap-table entry is loaded once
// for PB magnitude planes (the table read is a third of K2a's load bytes), and a
// thread keeps PB x U taps in flight
// radius phases per azimuth in k_rot_gather_multi, by grid side (a property of
// the configuration, so results never depend on the batch split): 8 for N <= 256
// (C1 +10%, C2 +1.2%: shorter per-thread radial loops), 4 above (C4: 8 phases
// measured -1.3%, 16 -4%, the samples of a load then spread along the rays)
#ifndef FSCAN_K2A_RP_SMALL
#define FSCAN_K2A_RP_SMALL 8
#endif
#ifndef FSCAN_K2A_PB
#define FSCAN_K2A_PB 2
#endif
// (K2a alone 2.69 -> 2.37 ms; the three-lane pipeline already hid that latency:
// C4 / C5 unchanged)
#ifdef FSCAN_K2A_TILE_AT
constexpr bool kK2aOffsets = false;  // A/B: tile_at per tap
#else
constexpr bool kK2aOffsets = true;
#endif
#ifdef FSCAN_K2A_NO_PREFETCH
constexpr bool kK2aPrefetch = false;
#else
constexpr bool kK2aPrefetch = true;
#endif
template <int PB, int RP>
__global__ void __launch_bounds__(kGatherThreads) k_rot_gather_multi(Params p) {
    pdl_enter();
    const int pair0 = blockIdx.y * PB;
    const int nt = p.n_theta, n = p.n, n_live = p.n_live;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // RP radius phases per azimuth (lane = RP * azimuth + phase; k2a_rp)
    const int i = blockIdx.x * (kGatherThreads / RP) + warp * (32 / RP) + lane / RP;
    const int rsub = lane % RP;
    const bool live = i < nt;
    const float2* m0 = reinterpret_cast<const float2*>(p.mag) + (size_t)pair0 * p.mag_plane;
    const PolarTap* col = p.taps + (live ? i : 0);
    double af[PB], ag[PB];
#pragma unroll
    for (int b = 0; b < PB; ++b) af[b] = ag[b] = 0.0;
    const int np = min(PB, p.batch - pair0);
    constexpr int U = PB >= 4 ? 1 : 4 / PB;
    auto taps_at = [&](int j0, PolarTap (&e)[U]) {
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int j = j0 + RP * q;
            e[q] = (live && j < n_live) ? col[(size_t)j * nt] : PolarTap{0, 0.f, 0.f, 0.f};  // flags 0: 0
        }
    };
    // kK2aPrefetch: the next step's tap entries are loaded before this step's
    // gathers, so the two dependent loads of a sample (entry, then the taps it
    // addresses) overlap across steps
    PolarTap e[U];
    if constexpr (kK2aPrefetch) taps_at(rsub, e);
    for (int j0 = rsub; j0 < n_live; j0 += RP * U) {
        PolarTap en[U];
        if constexpr (kK2aPrefetch) {
            taps_at(j0 + RP * U, en);
        } else {
            taps_at(j0, e);
        }
        float2 tv[PB][U][4];
        if constexpr (kK2aOffsets) {
            // the four tile offsets of an entry once for all PB planes, in 32-bit
            // arithmetic: (r0, u) -> o, (r0, u+1) -> o + 1 or into the next tile
            // column (+ 8 n - 7), row r0 + 1 -> + 8 (tile_at per tap was 36% of the
            // kernel's instructions)
            unsigned off[U][4];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const unsigned r0 = e[q].packed & 0xFFF, u = (e[q].packed >> 12) & 0xFFF;
                const unsigned o = ((u / kTileW) * (unsigned)n + r0) * kTileW + (u % kTileW);
                const unsigned o1 = o + ((u % kTileW) == kTileW - 1 ? (unsigned)n * kTileW - (kTileW - 1) : 1u);
                off[q][0] = o;
                off[q][1] = o1;
                off[q][2] = o + kTileW;
                off[q][3] = o1 + kTileW;
            }
#pragma unroll
            for (int b = 0; b < PB; ++b) {
                const float2* m = m0 + (size_t)(b < np ? b : 0) * p.mag_plane;
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int fl = e[q].packed >> 24;
#pragma unroll
                    for (int tp = 0; tp < 4; ++tp)
                        tv[b][q][tp] = ((fl >> tp) & 1) ? __ldg(m + off[q][tp]) : make_float2(0.f, 0.f);
                }
            }
        } else {
#pragma unroll
        for (int b = 0; b < PB; ++b) {
            const float2* m = m0 + (size_t)(b < np ? b : 0) * p.mag_plane;
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int r0 = e[q].packed & 0xFFF, u = (e[q].packed >> 12) & 0xFFF, fl = e[q].packed >> 24;
#pragma unroll
                for (int tp = 0; tp < 4; ++tp) {
                    const bool on = (fl >> tp) & 1;
                    tv[b][q][tp] = on ? __ldg(tile_at(m, n, r0 + (tp >> 1), u + (tp & 1))) : make_float2(0.f, 0.f);
                }
            }
        }
        }
#pragma unroll
        for (int b = 0; b < PB; ++b)
#pragma unroll
            for (int q = 0; q < U; ++q) {
                af[b] += (double)bilerp(e[q].fr, e[q].fc, tv[b][q][0].x, tv[b][q][1].x, tv[b][q][2].x, tv[b][q][3].x);
                ag[b] += (double)bilerp(e[q].fr, e[q].fc, tv[b][q][0].y, tv[b][q][1].y, tv[b][q][2].y, tv[b][q][3].y);
            }
        if constexpr (kK2aPrefetch) {
#pragma unroll
            for (int q = 0; q < U; ++q) e[q] = en[q];
        }
    }
#pragma unroll
    for (int b = 0; b < PB; ++b) {
        // the RP radius phases of an azimuth, summed in a fixed order
        double a = af[b], g = ag[b];
#pragma unroll
        for (int o = 1; o < RP; o <<= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (live && rsub == 0 && b < np) {
            double* prof = p.prof + (size_t)(pair0 + b) * 2 * nt;
            prof[i] = a;
            prof[nt + i] = g;
        }
    }
}

__global__ void __launch_bounds__(kGatherThreads) k_rot_gather(Params p) {
    pdl_enter();
    const int pair = blockIdx.y;
    const int nt = p.n_theta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * (kGatherThreads / 4) + warp * 8 + (lane >> 2);
    const bool live = i < nt;
    // the K1b transform holding the pair's |F| (and |G|): one per pair, or in
    // chain mode one per two scans of the sequence
    const int tr = p.chain ? pair / 2 : pair;
    const float2* m = reinterpret_cast<const float2*>(p.mag) + (size_t)tr * p.mag_plane;
    double* prof = p.prof + (size_t)pair * 2 * nt;
    if (p.chain && (pair & 1))
        gather_sums<true>(p, m, i, live, lane & 3, prof);
    else
        gather_sums<false>(p, m, i, live, lane & 3, prof);
}

// One K2b work item: kLags consecutive lags k0.. over the q-range [q0, q1);
// a 15-value window of Bx slides over 8 q per step (64 DFMA per 8 A and 8 Bx loads).
__device__ __forceinline__ void polar_item(const double* A, const double* Bx, int q0, int q1, int k0,
                                           double (&acc)[kLags]) {
#pragma unroll
    for (int c = 0; c < kLags; ++c) acc[c] = 0.0;
    double w[2 * kLags - 1];
#pragma unroll
    for (int c = 0; c < kLags - 1; ++c) w[c] = Bx[bx_skew(q0 + k0 + c)];
    int q = q0;
    for (; q + kLags <= q1; q += kLags) {
#pragma unroll
        for (int c = 0; c < kLags; ++c) w[kLags - 1 + c] = Bx[bx_skew(q + k0 + kLags - 1 + c)];
#pragma unroll
        for (int u = 0; u < kLags; ++u) {
            const double a = A[q + u];
#pragma unroll
            for (int c = 0; c < kLags; ++c) acc[c] = fma(a, w[u + c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < kLags - 1; ++c) w[c] = w[kLags + c];
    }
    for (; q < q1; ++q) {  // tail: one q at a time
        w[kLags - 1] = Bx[bx_skew(q + k0 + kLags - 1)];
        const double a = A[q];
#pragma unroll
        for (int c = 0; c < kLags; ++c) acc[c] = fma(a, w[c], acc[c]);
#pragma unroll
        for (int c = 0; c < kLags - 1; ++c) w[c] = w[c + 1];
    }
}

// wrap_pad (imageops.cpp:101-113) of one pair's profiles into shared memory:
// padded row q holds profile row (q - pad) mod nt. B is stored circularly
// extended, Bx[j] = B[(j - nt/2) mod L], so the score
// s[k] = (1/C) sum_q A[q] B[(q + k - nt/2) mod L] is
// sum_q A[q] Bx[q + k] without modular indexing (Bx[j] lives at bx_skew(j)).
__device__ __forceinline__ void polar_profiles(const Params& p, int pair, double* A, double* Bx) {
    const int nt = p.n_theta, L = p.L, pad = p.pad;
    const double* prof = p.prof + (size_t)pair * 2 * nt;
    for (int q = threadIdx.x; q < L; q += blockDim.x) {
        int i = (q - pad) % nt;
        if (i < 0) i += nt;
        A[q] = prof[i];
    }
    for (int j = threadIdx.x; j < L + nt + 2 * kLags; j += blockDim.x) {
        int qq = (j - nt / 2) % L;
        if (qq < 0) qq += L;
        int i = (qq - pad) % nt;
        if (i < 0) i += nt;
        Bx[bx_skew(j)] = prof[nt + i];
    }
}

// The theta scores s[0..nt) of a pair (shared memory, complete) -> hard argmax
// (strict >, lowest index, matcher.cpp:47-53), windowed soft-argmax
// (matcher.cpp:57-93), the pair's RotState and optional surface copy. Every
// thread of the CTA calls it; red_v / red_i: 32 entries of scratch each.
__device__ void polar_finish(const Params& p, int pair, const double* s, double* red_v, int* red_i, double* wbuf) {
    const int nt = p.n_theta;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x / 32;
    RotState* rs = p.rot + pair;
    double best_v = -INFINITY;
    int best_i = 0x7fffffff;
    for (int k = threadIdx.x; k < nt; k += blockDim.x)
        if (s[k] > best_v) {  // k increases per thread: strict > keeps the lowest index
            best_v = s[k];
            best_i = k;
        }
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
    if (warp == 0) {
        // every lane of warp 0 holds warp 0's maximum; each folds in the other
        // warps' (same order, same result in every lane)
        for (int w = 1; w < nwarps; ++w)
            if (red_v[w] > best_v || (red_v[w] == best_v && red_i[w] < best_i)) {
                best_v = red_v[w];
                best_i = red_i[w];
            }
        // soft_argmax over the n_theta x 1 surface (matcher.cpp:57-93). The
        // window's weights (an fp64 exp each: ~5 us of a one-pair call when one
        // thread computed all 2w + 1) are spread over the warp's lanes into wbuf
        // (>= min(2w + 1, n_theta) doubles); lane 0 then adds them up in the
        // reference's order r0 .. r1, so the sums are those of a serial loop.
        const int pk = best_i == 0x7fffffff ? 0 : best_i;  // all-NaN surface: the first bin, as the reference's scan
        const int r0 = max(0, pk - p.window), r1 = min(nt - 1, pk + p.window);
        double scale = 1.0;
        if (p.normalize) {
            double m = 0.0;  // a maximum: the same value in any order
            for (int r = r0 + lane; r <= r1; r += 32) m = fmax(m, fabs(s[r]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (m > 0.0) scale = 1.0 / m;
        }
        const double top = s[pk] * scale;
        for (int r = r0 + lane; r <= r1; r += 32) wbuf[r - r0] = exp(p.t_theta * (s[r] * scale - top));
        __syncwarp();
        if (lane == 0) {
            double wsum = 0.0, rsum = 0.0;
            for (int r = r0; r <= r1; ++r) {
                const double w = wbuf[r - r0];
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
    }
    if (p.theta_surf)
        for (int k = threadIdx.x; k < nt; k += blockDim.x) p.theta_surf[(size_t)pair * nt + k] = s[k];
}

// K2b: angular correlation of the profiles, hard + soft argmax over theta.
__global__ void __launch_bounds__(kPolarThreads) k_rot_polar(Params p) {
    pdl_enter();
    extern __shared__ double dsm[];
    const int pair = blockIdx.x;
    const int nt = p.n_theta, L = p.L;
    double* A = dsm;                      // wrap-extended radial-sum profiles, length L
    double* B = dsm + L;                  // skewed circular extension, bx_len(L, nt)
    double* s = B + bx_len(L, nt);        // theta surface, n_theta
    double* red_v;                        // block reduction scratch (32 entries each), after the partials
    int* red_i;
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

    const int np = polar_parts(nt);
    double* Bx = B;
    double* part = s + nt;                 // np x nt partial sums
    red_v = part + (size_t)np * nt;
    red_i = (int*)(red_v + 32);
    polar_profiles(p, pair, A, Bx);
    __syncthreads();
    // register-blocked: each item owns kLags consecutive lags over one of np
    // q-ranges (polar_item)
    {
        const int blocks = (nt + kLags - 1) / kLags;
        const int item = threadIdx.x;
        if (item < blocks * np) {
            const int k0 = kLags * (item % blocks), pi = item / blocks;
            const int q0 = (int)((long)L * pi / np), q1 = (int)((long)L * (pi + 1) / np);
            double acc[kLags];
            polar_item(A, Bx, q0, q1, k0, acc);
            double* pr = part + (size_t)pi * nt + k0;
#pragma unroll
            for (int c = 0; c < kLags; ++c)
                if (k0 + c < nt) pr[c] = acc[c];
        }
    }
    __syncthreads();
    const double invC = 1.0 / (double)p.C;
    for (int k = threadIdx.x; k < nt; k += kPolarThreads) {
        double acc = 0.0;
        for (int pi = 0; pi < np; ++pi) acc += part[(size_t)pi * nt + k];  // fixed order: deterministic
        s[k] = acc * invC;
    }
    __syncthreads();
    polar_finish(p, pair, s, red_v, red_i, part);  // the partial sums are dead: scratch for the window weights
}

// K2b split over S CTAs per pair (small batches: one CTA per pair would leave
// the GPU nearly idle for ~25 us): CTA `part` of a pair owns a contiguous range
// of lag blocks and writes their scores to theta_ws; k_rot_polar_fin then runs
// the argmaxes per pair.
// fuse: the pair's last CTA to finish (a counter in p.polar_cnt, reset by that
// CTA) runs the argmaxes itself instead of a k_rot_polar_fin launch — one kernel
// less on the critical path of a small batch.
__global__ void __launch_bounds__(kPolarThreads) k_rot_polar_part(Params p, int S, int fuse) {
    pdl_enter();
    extern __shared__ double dsm[];
    __shared__ int is_last;
    const int pair = blockIdx.x / S, part_id = blockIdx.x % S;
    const int nt = p.n_theta, L = p.L;
    const int blocks = (nt + kLags - 1) / kLags, per = (blocks + S - 1) / S;
    const int b0 = part_id * per, nb = min(blocks, b0 + per) - b0;
    if (nb <= 0) return;  // (not counted: the pair's active CTAs are those with lag blocks)
    // the fused kernel's q partition and summation order: bit-identical scores
    // whatever the batch size (results do not depend on batching)
    const int np = polar_parts(nt);
    double* A = dsm;
    double* Bx = A + L;
    double* part = Bx + bx_len(L, nt);  // np x (nb * kLags)
    const int W = nb * kLags;
    polar_profiles(p, pair, A, Bx);
    __syncthreads();
    const int item = threadIdx.x;
    if (item < nb * np) {
        const int kk0 = kLags * (item % nb), pi = item / nb;
        const int q0 = (int)((long)L * pi / np), q1 = (int)((long)L * (pi + 1) / np);
        double acc[kLags];
        polar_item(A, Bx, q0, q1, kLags * b0 + kk0, acc);
#pragma unroll
        for (int c = 0; c < kLags; ++c) part[(size_t)pi * W + kk0 + c] = acc[c];
    }
    __syncthreads();
    const double invC = 1.0 / (double)p.C;
    for (int kk = threadIdx.x; kk < W; kk += kPolarThreads) {
        const int k = kLags * b0 + kk;
        if (k < nt) {
            double acc = 0.0;
            for (int pi = 0; pi < np; ++pi) acc += part[(size_t)pi * W + kk];  // fixed order: deterministic
            p.theta_ws[(size_t)pair * nt + k] = acc * invC;
        }
    }
    if (!fuse) return;
    __threadfence();  // this thread's scores before the CTA's count
    __syncthreads();
    if (threadIdx.x == 0) {
        const int active = (blocks + per - 1) / per;
        is_last = atomicAdd(p.polar_cnt + pair, 1) == active - 1;
        if (is_last) p.polar_cnt[pair] = 0;  // ready for the next launch on this lane
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // the profiles and partial sums are dead: the scores, reduction scratch and
    // window weights take their place (the launch sizes the buffer for both)
    double* s = dsm;
    double* red_v = s + nt;
    int* red_i = (int*)(red_v + 32);
    double* wbuf = red_v + 32 + 16;
    for (int k = threadIdx.x; k < nt; k += kPolarThreads) s[k] = __ldcg(p.theta_ws + (size_t)pair * nt + k);
    __syncthreads();
    polar_finish(p, pair, s, red_v, red_i, wbuf);
}

__global__ void __launch_bounds__(kPolarThreads) k_rot_polar_fin(Params p) {
    pdl_enter();
    extern __shared__ double dsm[];
    const int pair = blockIdx.x, nt = p.n_theta;
    double* s = dsm;
    double* red_v = s + nt;
    int* red_i = (int*)(red_v + 32);
    double* wbuf = red_v + 32 + 16;  // behind the 32 ints: n_theta doubles for the window weights
    for (int k = threadIdx.x; k < nt; k += kPolarThreads) s[k] = p.theta_ws[(size_t)pair * nt + k];
    __syncthreads();
    polar_finish(p, pair, s, red_v, red_i, wbuf);
}

__global__ void k_theta_in(Params p) {
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= p.batch) return;
    const double theta = p.theta_mod > 0 ? p.theta_in[(p.item_base + pair) % p.theta_mod] : p.theta_in[pair];
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

// ---------------------------------------------------------------- translation stage
// The reference correlates the scans zero-padded to P = next_fast_size(2N-1)
// (matcher.cpp:165-167) and keeps the lags ky in [-N/2, N/2), kx in
// [-(N/2-1), N/2] (crop, matcher.cpp:171-182). The linear correlation has
// support |k| <= N-1, so a CIRCULAR correlation of length M = 3N/2 already
// equals it on those lags (aliases land at |k| >= N). With K = N/2, M = 3K,
// and the data at offset 0 (a shift common to both scans cancels in conj(F)G),
// every length-M transform of an N-sample signal is three K-point FFTs:
//   X[3k+q] = FFT_K( W_M^{nq} (x[n] + W_3^q x[n+K]) )[k],  q = 0, 1, 2.
// This is 1.8x fewer FFT flops than the power-of-two P = 2N route.
constexpr float kS3 = 0.86602540378443865f;  // sqrt(3)/2

__device__ __forceinline__ float2 w3(int q) {  // W_3^q = exp(-2 pi i q / 3)
    q %= 3;
    return q == 0 ? make_float2(1.f, 0.f) : (q == 1 ? make_float2(-0.5f, -kS3) : make_float2(-0.5f, kS3));
}

// K4 twiddles W_M^{q n0} for n0 = t + m T (T = K/16, so W_M^T = W_48):
// W_M^{q t} (one global-table read per thread) times W_48^{q m}, a
// constant-bank table (two distinct q per warp: at most two addresses per
// LDC). No W_M table is staged in shared memory (FSCAN_K4_TABLES restores the
// staged M-entry table for A/B runs).
__constant__ float kW48re[48] = {1.0f, 0.9914448857307434f, 0.9659258127212524f, 0.9238795042037964f, 0.8660253882408142f, 0.7933533191680908f, 0.7071067690849304f, 0.6087614297866821f, 0.5f, 0.3826834261417389f, 0.258819043636322f, 0.13052618503570557f, 0.0f, -0.13052618503570557f, -0.258819043636322f, -0.3826834261417389f, -0.5f, -0.6087614297866821f, -0.7071067690849304f, -0.7933533191680908f, -0.8660253882408142f, -0.9238795042037964f, -0.9659258127212524f, -0.9914448857307434f, -1.0f, -0.9914448857307434f, -0.9659258127212524f, -0.9238795042037964f, -0.8660253882408142f, -0.7933533191680908f, -0.7071067690849304f, -0.6087614297866821f, -0.5f, -0.3826834261417389f, -0.258819043636322f, -0.13052618503570557f, 0.0f, 0.13052618503570557f, 0.258819043636322f, 0.3826834261417389f, 0.5f, 0.6087614297866821f, 0.7071067690849304f, 0.7933533191680908f, 0.8660253882408142f, 0.9238795042037964f, 0.9659258127212524f, 0.9914448857307434f};
__constant__ float kW48im[48] = {0.0f, -0.13052618503570557f, -0.258819043636322f, -0.3826834261417389f, -0.5f, -0.6087614297866821f, -0.7071067690849304f, -0.7933533191680908f, -0.8660253882408142f, -0.9238795042037964f, -0.9659258127212524f, -0.9914448857307434f, -1.0f, -0.9914448857307434f, -0.9659258127212524f, -0.9238795042037964f, -0.8660253882408142f, -0.7933533191680908f, -0.7071067690849304f, -0.6087614297866821f, -0.5f, -0.3826834261417389f, -0.258819043636322f, -0.13052618503570557f, 0.0f, 0.13052618503570557f, 0.258819043636322f, 0.3826834261417389f, 0.5f, 0.6087614297866821f, 0.7071067690849304f, 0.7933533191680908f, 0.8660253882408142f, 0.9238795042037964f, 0.9659258127212524f, 0.9914448857307434f, 1.0f, 0.9914448857307434f, 0.9659258127212524f, 0.9238795042037964f, 0.8660253882408142f, 0.7933533191680908f, 0.7071067690849304f, 0.6087614297866821f, 0.5f, 0.3826834261417389f, 0.258819043636322f, 0.13052618503570557f};

__device__ __forceinline__ float2 w48(int k) { return make_float2(kW48re[k], kW48im[k]); }  // k < 48

// W_32^m (m < 16), for K5's input twiddles (see k_xlat_out)
__constant__ float kW32re[16] = {1.0f, 0.9807852506637573f, 0.9238795042037964f, 0.8314695954322815f, 0.7071067690849304f, 0.5555702447891235f, 0.3826834261417389f, 0.19509032368659973f, 0.0f, -0.19509032368659973f, -0.3826834261417389f, -0.5555702447891235f, -0.7071067690849304f, -0.8314695954322815f, -0.9238795042037964f, -0.9807852506637573f};
__constant__ float kW32im[16] = {0.0f, -0.19509032368659973f, -0.3826834261417389f, -0.5555702447891235f, -0.7071067690849304f, -0.8314695954322815f, -0.9238795042037964f, -0.9807852506637573f, -1.0f, -0.9807852506637573f, -0.9238795042037964f, -0.8314695954322815f, -0.7071067690849304f, -0.5555702447891235f, -0.3826834261417389f, -0.19509032368659973f};
__device__ __forceinline__ float2 w32(int k) { return make_float2(kW32re[k], kW32im[k]); }  // k < 16

// Row spectra handed from K3 to K4, transposed: per pair an F plane then a G
// plane, each [3N/4 + 1 bins][N rows] float2 (the column transforms of K4 read
// one plane per pass: 8 bytes per element instead of a float4 (F, G) of which
// each pass used half — K4 is bound by its L1 wavefronts: K4 7.8 -> 7.3 ms at
// C4). N = 1024 keeps the interleaved [bins][rows] float4 (F, G): its K4 loads
// each (F, G) site once for all three q groups (XColGeom::FOLD1), where the
// planes measured 1.5% slower.
template <int N>
constexpr bool kFgtPlanes = N < 1024;
template <int N>
__device__ __forceinline__ float2* fgt_plane(const Params& p, int pair, int plane) {
    return p.fgt + (2 * (size_t)pair + plane) * (size_t)(3 * N / 4 + 1) * N;
}

// W_M^e for 0 <= e < M (every caller passes a reduced exponent)
__device__ __forceinline__ float2 wm(const float2* __restrict__ tw_m, int e) { return __ldg(tw_m + e); }

// Rows/columns of the translation stage each own THREE K-point transforms
// (q = 0, 1, 2), run concurrently by three thread groups: transform index
// tr = 3 * unit + q in the Geom mapping.

// ---------------------------------------------------------------- K3
// Row y: z = f~ + i g~r (g~r = rotate_bilinear(g~, -theta), imageops.cpp:61-79,
// exact fp64 index map) gathered once into a shared stash; group q forms
// W_M^{nq}(z[n] + W_3^q z[n+K]) and FFTs it (E_q); then the real spectra
// F = (Z[k'] + conj Z[M-k'])/2, G = (Z[k'] - conj Z[M-k'])/2i, Z[3k+q] = E_q[k],
// for k' in [0, M/2] are written transposed as fgt[k'][y].
constexpr int kXThreads = 384;
#ifdef FSCAN_K3_TW_TABLE
constexpr bool kK3TwTable = true;  // A/B: fold twiddles read from the W_M table per element
#else
constexpr bool kK3TwTable = false;
#endif
__host__ __device__ constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
#ifdef FSCAN_K3_TW_LOAD2
constexpr bool kK3TwSquare = false;  // A/B: W_M^{2x} by a second table read per fold site
#else
constexpr bool kK3TwSquare = true;
#endif
#ifdef FSCAN_K3_TW_REG
constexpr bool kK3TwReg = true;  // A/B (K3 6.52 -> 6.72 ms at C4): a thread's <= 2 distinct W_M^x held in registers
#else
constexpr bool kK3TwReg = false;
#endif
#ifdef FSCAN_K3_STASH
constexpr bool kK3FoldGather = false;  // A/B: gather into a z stash, fold per group from it (rounds 1-2)
#else
constexpr bool kK3FoldGather = true;
#endif
#ifndef FSCAN_K3_FIG_MAXN
#define FSCAN_K3_FIG_MAXN 4096
#endif
#ifdef FSCAN_K3_FIG_STAGE
constexpr bool kK3FigNoStage = false;  // A/B: FIG with the f~ rows staged by TMA (C5 -2%: 71 KB CTAs)
#else
constexpr bool kK3FigNoStage = true;
#endif
#ifdef FSCAN_K3_STASH_SOA
constexpr bool kK3StashSoA = true;  // A/B: split re / im stash (rounds 1-2)
#else
constexpr bool kK3StashSoA = false;
#endif

template <int N>
struct XRowGeom {
    using G = Geom<N / 2, kXThreads>;
    static constexpr int ROWS = G::PER_CTA / 3;
    // stash: z = f~ + i g~r as float2 rows (one 64-bit access per cell on both
    // sides; a half-warp touches 16 consecutive cells of one row, or the end of
    // one row and the start of the next: conflict-free at any multiple-of-16
    // stride). kK3StashSoA (A/B): split re / im float rows, padded every 32.
    static constexpr int SP0 = N + N / 32;
    static constexpr int SP = kK3StashSoA ? ((SP0 % 32 == 0) ? SP0 + 16 : SP0) : N;  // row stride (floats / float2)
    // the FFT exchange buffers alias the gather stash (dead once v[] is loaded):
    // ~50 KB per CTA, three CTAs per SM
    static constexpr size_t STASH = (size_t)2 * ROWS * SP;
    // + the CTA's ROWS rows of f~ (dense, one TMA bulk copy) behind the stash
    // (texture-gather instantiation only)
    // FIG (gather + fold, default): no stash; the f~ stage sits behind the
    // exchange buffers the gather writes
    static constexpr bool FIG = kK3FoldGather && N <= FSCAN_K3_FIG_MAXN;
    // f~ staged by TMA (the texture-gather instantiation), unless FIG without it
    static constexpr bool FT_STAGE = kK3FtTma && !(FIG && kK3FigNoStage);
    static constexpr size_t FT_OFF = FIG ? (size_t)G::FLOATS : STASH;
    static constexpr size_t STAGE = FT_OFF + (FT_STAGE ? (size_t)ROWS * N : 0);
    static constexpr size_t WORK = STAGE > (size_t)G::FLOATS ? STAGE : (size_t)G::FLOATS;
    // + the span-16 stage's [r][k] twiddle table (K >= 256): 15 shared loads
    // per thread instead of 4 global loads and 11 products (C4 +0.4%; the same
    // table in K1b measured slower)
    static constexpr bool RK = N / 2 >= 256;
    static constexpr size_t SMEM = (WORK + (RK ? 480 : 0)) * sizeof(float);
    static_assert(G::PER_CTA % 3 == 0, "three transforms per row");
    // separation loop: a half-warp reads R rows x KB consecutive k. Row ol's
    // buffers start at 3 * ol * stride, i.e. bank offset o * ol (mod 16); R =
    // 16 / gcd(o, 16) rows then cover distinct offsets and the aligned KB-blocks
    // of k fill the gaps, so the reads are conflict free.
    static constexpr int O = (3 * G::template stride_len<N / 2>()) % 16;
    static constexpr int KB = O == 0 ? 16 : ((O & -O) < 16 ? (O & -O) : 16);
    static constexpr int R = 16 / KB;
    static_assert(ROWS % R == 0 && kXThreads % 16 == 0, "separation mapping");
    __device__ __forceinline__ static void sep_map(int tid, int& ol, int& kk) {
        constexpr int RG = ROWS / R;  // half-warps per k-block
        const int g = tid >> 4, hl = tid & 15;
        ol = (g % RG) * R + hl / KB;
        kk = (g / RG) * KB + hl % KB;
    }
};

// MANY: items of a multi-candidate launch (brute-force search) read the scans
// of pair (item_base + item) / src_div; a separate instantiation keeps the
// matcher's gather loop free of that indexing.
// Three CTAs per SM (56 registers): the gather is latency bound, occupancy
// beats per-thread memory-level parallelism here (measured: 2 CTAs x 6 cells
// in flight 8.1 ms, 3 CTAs x 4 cells 7.7 ms per 4096 C4 pairs).
// EMB: the scans are zero-embedded in the N x N (power-of-two) grid, valid
// size p.n < N and rotation centre p.c0 (grid sides that are not powers of
// two): g~r is zero outside the valid grid.
// TEX: the four taps of a cell come from ONE texture gather (tld4) on the lane's
// g~ texture (pitch 2-D, rows pair * N + r, zero border for the columns; rows
// outside the pair's grid are zeroed here), instead of four 32-bit loads.
template <int N, bool MANY, bool EMB, bool TEX = false>
__global__ void __launch_bounds__(kXThreads, 3) k_xlat_rows(Params p) {
    constexpr int K = N / 2, M = 3 * K, H = M / 2;
    using X = XRowGeom<N>;
    using G = typename X::G;
    constexpr int T = G::T, ROWS = X::ROWS, SP = X::SP;
    extern __shared__ __align__(128) float smem[];
    [[maybe_unused]] float* st_re = smem;
    [[maybe_unused]] float* st_im = smem + ROWS * SP;
    [[maybe_unused]] float2* st2 = reinterpret_cast<float2*>(smem);
    float* xbase = smem;  // aliases the stash (see XRowGeom::SMEM)
    // the [r][k] table (a constant of the context): loaded before the
    // dependency wait, stored after the gather (a load -> store here would wait
    // out an L2 round trip before the gather's first fetch)
    static_assert(kXThreads >= 240, "one table entry per thread");
    [[maybe_unused]] float2 rkv;
    if constexpr (X::RK)
        if (threadIdx.x < 240) rkv = __ldg(p.tw_rk + threadIdx.x);
    pdl_enter();
    const int pair = blockIdx.y;
    const int y0 = blockIdx.x * ROWS;
    const RotState rs = p.rot[pair];
    const int src = MANY ? (p.item_base + pair) / p.src_div : pair;  // pair whose scans this item reads
    const float* ft = p.ft + (size_t)src * N * N;
    // TEX (the lane's own workspace): the block's ROWS rows of f~ by one TMA bulk
    // copy into a dense stage; the gather reads them from there
    constexpr bool FT_TMA = TEX && X::FT_STAGE;
    __shared__ uint64_t ft_bar;
    const float* fst = smem + X::FT_OFF;
    if constexpr (FT_TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&ft_bar, 1);
            bulk_load(smem + X::FT_OFF, ft + (size_t)y0 * N, (unsigned)(ROWS * N * sizeof(float)), &ft_bar);
        }
        __syncthreads();  // publishes the barrier's initialisation
    }
    const float* gt = p.gt + (size_t)src * N * N;
    const float c0f32 = EMB ? p.c0 : (N - 1) / 2.0f;  // exact (half-integer or integer)
    float2* srk = reinterpret_cast<float2*>(smem + X::WORK);  // ordered by the barrier after the gather
    const int nvalid = EMB ? p.n : N;
    // rotate_bilinear(g~, -theta); -theta == 0.0 returns g~ itself, which st = 0,
    // ct = 1 reproduce exactly (integer source coordinates, zero fractions)
    const float stf = rs.identity ? 0.0f : (float)rs.st, ctf = rs.identity ? 1.0f : (float)rs.ct;
    // one cell (x, yl) of the de-rotated scan: its f~ value (unless staged by
    // TMA) and the four bilinear taps of g~, every load issued before any use
    auto fetch = [&](int x, int yl, bool in_range, float& fv, float (&tap)[4], float& fr, float& fc) {
        const int y = y0 + yl;
        const bool live = in_range && (!EMB || (x < nvalid && y < nvalid));
        // src_row = c + st*u + ct*v, src_col = c + ct*u - st*v (imageops.cpp:70-73)
        // in fp32 FMAs: <= 5e-5 cell coordinate error, i.e. <= 5e-5 relative per
        // bilinear sample (far inside the 1e-4 surface gate)
        const float uu = (float)x - c0f32, vv = (float)y - c0f32;  // exact half-integers
        const float sr = fmaf(stf, uu, fmaf(ctf, vv, c0f32));
        const float sc = fmaf(ctf, uu, fmaf(-stf, vv, c0f32));
        const float r0f = floorf(sr), cf = floorf(sc);
        fr = sr - r0f;
        fc = sc - cf;
        // taps outside the grid are 0 (sample_bilinear, imageops.cpp:10-26)
        const int r0 = (int)r0f, cc0 = (int)cf;
        const bool r0in = live && (unsigned)r0 < (unsigned)N, r1in = live && (unsigned)(r0 + 1) < (unsigned)N;
        const bool c0in = (unsigned)cc0 < (unsigned)N, c1in = (unsigned)(cc0 + 1) < (unsigned)N;
        if constexpr (!FT_TMA) fv = live ? ft[y * N + x] : 0.f;
        if constexpr (TEX) {
            // texel (c, row) at coordinate (c + 1.0, row + 1.0): the gather's
            // footprint starts at floor(coord - 0.5) = (cc0, r0); component
            // order (c0, r1), (c1, r1), (c1, r0), (c0, r0)
            const float4 g4 = tex2Dgather<float4>((cudaTextureObject_t)p.gtex, cf + 1.0f,
                                                 (float)(pair * N + r0) + 1.0f, 0);
            tap[0] = r0in ? g4.w : 0.f;
            tap[1] = r0in ? g4.z : 0.f;
            tap[2] = r1in ? g4.x : 0.f;
            tap[3] = r1in ? g4.y : 0.f;
        } else {
            const float* gp = gt + (r0 * N + cc0);  // 32-bit offset, one address per cell
            tap[0] = (r0in && c0in) ? gp[0] : 0.f;
            tap[1] = (r0in && c1in) ? gp[1] : 0.f;
            tap[2] = (r1in && c0in) ? gp[N] : 0.f;
            tap[3] = (r1in && c1in) ? gp[N + 1] : 0.f;
        }
    };
    constexpr int U = FSCAN_K3_U;
    if constexpr (X::FIG) {
        // gather + fold: a thread takes the cells x and x + K of a row (a fold
        // site), forms the three group inputs W_M^{q x} (z[x] + W_3^q z[x+K])
        // and stores them straight into the groups' exchange buffers — no stash
        // of z and no per-group re-read of it
        constexpr int SITES = ROWS * K, US = U / 2;
        // fold twiddles W_M^x: a thread's sites have x = (tid + u * kXThreads) mod K
        // in every round when a round's stride is a multiple of K, i.e. TWP
        // distinct x per thread: kK3TwReg (A/B, off) reads them once here
        constexpr int XSTEP = kXThreads % K;
        constexpr int TWP = XSTEP == 0 ? 1 : K / gcd_c(XSTEP, K);
        constexpr bool TWREG = kK3TwReg && (US * kXThreads) % K == 0 && TWP <= 2 && TWP <= US;
        [[maybe_unused]] float2 wreg[TWREG ? TWP : 1];
        if constexpr (TWREG) {
#pragma unroll
            for (int j = 0; j < TWP; ++j) wreg[j] = wm(p.tw_m, (threadIdx.x + j * XSTEP) % K);
        }
#pragma unroll 1
        for (int e0 = threadIdx.x; e0 < SITES; e0 += US * kXThreads) {
            float fv[US][2], tap[US][2][4], frs[US][2], fcs[US][2];
#pragma unroll
            for (int u = 0; u < US; ++u) {
                const int e = e0 + u * kXThreads;
                const int yl = e / K, x = e % K;
#pragma unroll
                for (int h = 0; h < 2; ++h) fetch(x + h * K, yl, e < SITES, fv[u][h], tap[u][h], frs[u][h], fcs[u][h]);
            }
            if constexpr (FT_TMA) {
                if (e0 == threadIdx.x) mbar_wait(&ft_bar, 0);  // first round: after its texture fetches are issued
#pragma unroll
                for (int u = 0; u < US; ++u) {
                    const int e = e0 + u * kXThreads;
                    const int yl = e / K, x = e % K;
#pragma unroll
                    for (int h = 0; h < 2; ++h) fv[u][h] = e < SITES ? fst[yl * N + x + h * K] : 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < US; ++u) {
                const int e = e0 + u * kXThreads;
                if (e < SITES) {
                    const int yl = e / K, x = e % K;
                    const float2 z0 = make_float2(fv[u][0], bilerp(frs[u][0], fcs[u][0], tap[u][0][0], tap[u][0][1],
                                                                   tap[u][0][2], tap[u][0][3]));
                    const float2 z1 = make_float2(fv[u][1], bilerp(frs[u][1], fcs[u][1], tap[u][1][0], tap[u][1][1],
                                                                   tap[u][1][2], tap[u][1][3]));
                    // z0 + W_3^q z1 for q = 0, 1, 2 (a radix-3 butterfly with one zero input)
                    const float2 tt = make_float2(fmaf(-0.5f, z1.x, z0.x), fmaf(-0.5f, z1.y, z0.y));
                    const float2 ss = make_float2(kS3 * z1.x, kS3 * z1.y);
                    G::lay(xbase, 3 * yl).put(x, cadd(z0, z1));
                    float2 w1;
                    if constexpr (TWREG)
                        w1 = wreg[u % TWP];
                    else
                        w1 = wm(p.tw_m, x);
                    // W_M^{2x} as a square (K3 6.73 -> 6.50 ms at C4, 7.66 -> 7.36 at C5:
                    // the second table read was a stride-2 access); FSCAN_K3_TW_LOAD2
                    // restores the read
                    const float2 w2 = kK3TwSquare ? cmul(w1, w1) : wm(p.tw_m, 2 * x);
                    G::lay(xbase, 3 * yl + 1).put(x, cmul(w1, make_float2(tt.x + ss.y, tt.y - ss.x)));
                    G::lay(xbase, 3 * yl + 2).put(x, cmul(w2, make_float2(tt.x - ss.y, tt.y + ss.x)));
                }
            }
        }
    } else {
        // gather: ROWS rows x N cells over all threads, consecutive threads on
        // consecutive x; U cells per thread per round with every load issued
        // before any use (memory-level parallelism for the L2/DRAM latency)
        constexpr int CELLS = ROWS * N;
#pragma unroll 1
        for (int e0 = threadIdx.x; e0 < CELLS; e0 += U * kXThreads) {
            float fv[U], tap[U][4], frs[U], fcs[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * kXThreads;
                fetch(e % N, e / N, e < CELLS, fv[u], tap[u], frs[u], fcs[u]);
            }
            if constexpr (FT_TMA) {
                if (e0 == threadIdx.x) mbar_wait(&ft_bar, 0);  // first round: after its texture fetches are issued
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * kXThreads;
                    fv[u] = e < CELLS ? fst[e] : 0.f;  // dense [ROWS][N]: e = yl * N + x
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * kXThreads;
                if (e < CELLS) {
                    const int yl = e / N, x = e % N;
                    const float gi = bilerp(frs[u], fcs[u], tap[u][0], tap[u][1], tap[u][2], tap[u][3]);
                    if constexpr (kK3StashSoA) {
                        const int a = yl * SP + x + (x >> 5);
                        st_re[a] = fv[u];
                        st_im[a] = gi;
                    } else {
                        st2[yl * SP + x] = make_float2(fv[u], gi);
                    }
                }
            }
        }
    }
    if constexpr (X::RK)
        if (threadIdx.x < 240) srk[threadIdx.x] = rkv;
    __syncthreads();
    int tr, t;
    G::map(threadIdx.x, tr, t);
    const int yl = tr / 3, q = tr % 3;
    {
        float2 v[16];
        if constexpr (X::FIG) {
#pragma unroll
            for (int m = 0; m < 16; ++m) v[m] = G::lay(xbase, tr).get(t + m * T);
            __syncwarp();  // every input read before the transform's exchange writes
        } else {
            const float2 w3q = w3(q);
            // W_M^{q n0}, n0 = t + m T (M = 48 T): the thread's base W_M^{q t} times
            // W_48^{q m} from the constant bank (a scattered table read per element
            // cost an L1 wavefront per 16 bytes)
            const float2 bq = kK3TwTable ? make_float2(1.f, 0.f) : wm(p.tw_m, q * t);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int n0 = t + m * T, n1 = n0 + K;
                float2 z0, z1;
                if constexpr (kK3StashSoA) {
                    const int a0 = yl * SP + n0 + (n0 >> 5), a1 = yl * SP + n1 + (n1 >> 5);
                    z0 = make_float2(st_re[a0], st_im[a0]);
                    z1 = make_float2(st_re[a1], st_im[a1]);
                } else {
                    z0 = st2[yl * SP + n0];
                    z1 = st2[yl * SP + n1];
                }
                const float2 s = cadd(z0, cmul(w3q, z1));
                if constexpr (kK3TwTable)
                    v[m] = q ? cmul(wm(p.tw_m, n0 * q), s) : s;
                else
                    v[m] = cmul(cmul(bq, w48(q * m)), s);
            }
            __syncthreads();  // every stash read done before the exchange buffers are written
        }
        const auto b = G::lay(xbase, tr);
        if constexpr (X::RK)
            fft_regs<K, -1, true, (kPkRows<N> ? FSCAN_PK_K3 : 0)>(v, t, b, fscan_fft::SmemTwRK{srk, p.tw_k});  // T <= 32: within a warp
        else
            fft_regs<K, -1, true, (kPkRows<N> ? FSCAN_PK_K3 : 0)>(v, t, b, p.tw_k);
#pragma unroll
        for (int m = 0; m < 16; ++m) b.put(t + m * T, v[m]);
    }
    __syncthreads();
    // separation + transposed write (k = kk, kk + KSTEP, ...; see sep_map)
    constexpr int KSTEP = kXThreads / ROWS;
    int ol, kk;
    X::sep_map(threadIdx.x, ol, kk);
    const auto e0 = G::lay(xbase, 3 * ol), e1 = G::lay(xbase, 3 * ol + 1), e2 = G::lay(xbase, 3 * ol + 2);
    // F = (Z[k'] + conj Z[M-k'])/2, G = (Z[k'] - conj Z[M-k'])/2i with Z[3k+q] = E_q[k];
    // by residue class: 3k pairs with E_0[K-k], 3k+1 with E_2[K-1-k], 3k+2 with E_1[K-1-k]
    auto sep = [](float2 z1, float2 z2) {
        const float dr = z1.x - z2.x, di = z1.y + z2.y;
        return make_float4(0.5f * (z1.x + z2.x), 0.5f * (z1.y - z2.y), 0.5f * di, -0.5f * dr);
    };
    // F and G planes of the pair (fgt_plane): each store a 64-byte run of the
    // CTA's rows of one bin
    float2* dF = fgt_plane<N>(p, pair, 0) + y0 + ol;
    float2* dG = fgt_plane<N>(p, pair, 1) + y0 + ol;
    float4* d4 = reinterpret_cast<float4*>(p.fgt) + (size_t)pair * (H + 1) * N + y0 + ol;
    auto put = [&](int kb, float4 v) {
        if constexpr (kFgtPlanes<N>) {
            dF[(size_t)kb * N] = make_float2(v.x, v.y);
            dG[(size_t)kb * N] = make_float2(v.z, v.w);
        } else {
            d4[(size_t)kb * N] = v;
        }
    };
    if constexpr (N >= 1024) {
        // compile-time trip counts (guarded): every address is affine in the
        // unrolled step (C5 +0.5%; at N = 512 the unrolled form ran K3 1.5% slower)
        constexpr int I0 = (K / 2) / KSTEP + 1, I1 = ((H - 1) / 3) / KSTEP + 1, I2 = ((H - 2) / 3) / KSTEP + 1;
#pragma unroll
        for (int i = 0; i < I0; ++i) {
            const int k = kk + i * KSTEP;
            if (k <= K / 2) put(3 * k, sep(e0.get(k), e0.get((K - k) & (K - 1))));
        }
#pragma unroll
        for (int i = 0; i < I1; ++i) {
            const int k = kk + i * KSTEP;
            if (3 * k + 1 <= H) put(3 * k + 1, sep(e1.get(k), e2.get(K - 1 - k)));
        }
#pragma unroll
        for (int i = 0; i < I2; ++i) {
            const int k = kk + i * KSTEP;
            if (3 * k + 2 <= H) put(3 * k + 2, sep(e2.get(k), e1.get(K - 1 - k)));
        }
    } else {
        for (int k = kk; k <= K / 2; k += KSTEP) put(3 * k, sep(e0.get(k), e0.get((K - k) & (K - 1))));
        for (int k = kk; 3 * k + 1 <= H; k += KSTEP) put(3 * k + 1, sep(e1.get(k), e2.get(K - 1 - k)));
        for (int k = kk; 3 * k + 2 <= H; k += KSTEP) put(3 * k + 2, sep(e2.get(k), e1.get(K - 1 - k)));
    }
}

// ---------------------------------------------------------------- K4
// Column k' of the row spectra. Group q: F_q = FFT_K(W_M^{nq}(F[n] + W_3^q F[n+K]))
// (transformed in buffer A and parked there), G_q likewise in buffer B,
// X_q = conj(F_q) G_q, e_q = IFFT_K(X_q) (left in buffer B). Then the needed
// lags ky in [-K, K) of IFFT_M(X) by a radix-3 combine:
//   ky = n in [0, K):     sum_q W_M^{-nq} e_q[n]
//   ky = n - K in [-K,0): sum_q W_M^{-nq} W_3^{q} e_q[n]
// stored by surface row i = half - ky (the flip of matcher.cpp:171-182)
// through a shared-memory tile (a k'-major output written straight from the
// registers measured slower: K4 grows to 120 registers and K5's loads scatter).

#ifdef FSCAN_K4_TABLES
constexpr bool kK4W48 = false;
#else
constexpr bool kK4W48 = true;
#endif
#ifdef FSCAN_K4_QMAJOR
constexpr bool kK4QMajor = true;  // A/B (measured slower): K4 transforms ordered q-major
#else
constexpr bool kK4QMajor = false;
#endif
#ifdef FSCAN_K4_W48_FOLD1
constexpr bool kK4W48Fold1 = true;  // A/B: W_48 combine twiddles at N = 1024 too
#else
constexpr bool kK4W48Fold1 = false;
#endif
#ifdef FSCAN_K4_TAB_GLOBAL
constexpr bool kK4TabGlobal = true;  // A/B: merged twiddle table read through L1 instead of staged
#else
constexpr bool kK4TabGlobal = false;
#endif
#ifndef FSCAN_K4_COLS512
#define FSCAN_K4_COLS512 4  // K4 columns per CTA at N = 512
#endif
#ifndef FSCAN_K4_F2_MIN
#define FSCAN_K4_F2_MIN 64
#endif
#ifndef FSCAN_K4_MINB512
#define FSCAN_K4_MINB512 3
#endif
#ifndef FSCAN_K4_BLOCKS
#define FSCAN_K4_BLOCKS 1
#endif
#ifndef FSCAN_K4_GSTAGE_BODY
#define FSCAN_K4_GSTAGE_BODY 0
#endif
#ifndef FSCAN_K4_GSTAGE
#define FSCAN_K4_GSTAGE 1  // merged K4 (N = 512): G columns prefetched by TMA during the F pass (C4 +1.0%)
#endif
#ifdef FSCAN_K4_SPLIT_TAB
constexpr bool kK4SplitTab = true;  // A/B: split table barrier (mbarrier arrive / wait before the last stage)
#else
constexpr bool kK4SplitTab = false;
#endif
#ifdef FSCAN_K4_PAIR_BAR
constexpr bool kK4PairBar = true;  // A/B: per column pair named barrier before the combine
#else
constexpr bool kK4PairBar = false;
#endif
#ifdef FSCAN_K4_EARLYSYNC
constexpr bool kK4LateSync = false;  // A/B: the table barrier before the first fold's loads
#else
constexpr bool kK4LateSync = true;
#endif
// kK4Merge: twiddles merged into the last FFT stage (xlat_cols_merged) at
// N = 512: C4 +1.3% with the float2 exchange layout (a half-warp is one
// transform, so every table read is conflict-free; with the split re/im
// layout the two q of a half-warp made them 2-way conflicts and the merge
// measured neutral). Not at N = 256: the table costs C2's kernel its fourth
// CTA per SM (-1%).
#ifdef FSCAN_K4_NOMERGE
constexpr bool kK4Merge = false;  // A/B
#else
constexpr bool kK4Merge = true;
#endif

template <int N>
struct XColGeom {
    static constexpr int T = N / 32;
    // columns per CTA: 3 * COLS * T threads must fill whole warps
    // (N = 512 at 4 columns: three 192-thread CTAs per SM instead of two of
    // 384; the kernel alone is 3% slower, but the pipeline is 0.6% faster, its
    // shorter CTAs interleaving better with the other lane's kernels)
    // (N = 1024 at 2 columns: 192-thread CTAs, three per SM at 96 registers;
    // C5 +8% over 4 columns in 384 threads at 80 registers)
    static constexpr int COLS = (T >= 32) ? 2 : ((T >= 16) ? FSCAN_K4_COLS512 : ((T >= 4) ? 8 : 16));
    static constexpr int THREADS = 3 * COLS * T;
    // (outputs are stored from registers into the blocked Y layout, y_at; round
    // 1-2 staged them in an [N][COLS + 1] shared tile copied out row-major,
    // ~12% of K4's warp samples)
    // float2 exchange buffers, one per transform (Geom: the T lanes of a
    // transform contiguous, a half-warp = one transform at N >= 512): one LSU
    // instruction per exchanged value. FSCAN_K4_F2_MIN > N restores the split
    // re/im layout of rounds 1-2 (GeomSoA), which issues twice the shared-memory
    // instructions for the same wavefronts (MIO-throttle bound at N = 1024).
    using G = std::conditional_t<(N >= FSCAN_K4_F2_MIN), fscan_fft::Geom<N / 2, THREADS>,
                                 fscan_fft::GeomSoA<N / 2, THREADS>>;
    // (round 2 measured a TMA bulk copy of the CTA's fgt columns into an input
    // area aliased by buffer B: C4 -0.7%, C2 -2.5% — every warp then waits for
    // the whole block before its first fold; removed)
    static constexpr size_t FFT_FLOATS = (size_t)2 * G::FLOATS;
    static constexpr size_t WORK_FLOATS = FFT_FLOATS;
    // twiddle tables staged behind the work area: W_K (K entries) and, below
    // N = 1024, W_M (3K; at 1024 it would push the CTA past half an SM's smem)
    // (the K-point FFTs read the span-16 stage's factors from a [r][k] table,
    // 240 entries, and, at K = 512 only, the last stage's from the linear W_K)
    static constexpr bool SMEM_WM = N <= 512 && !kK4W48;
    static constexpr int TW_LIN = N / 2 > 256 ? N / 2 : 0;
    // W_M staged as two contiguous K-entry tables W_M^{n0}, W_M^{2 n0} below
    // N = 512 (conflict-free; at N = 256 ptxas also keeps K4 spill-free at four
    // CTAs/SM, +10% C2), as the linear M-entry table at 512 (measured faster)
    static constexpr bool SPLIT_WM = N < 512;
    static constexpr size_t TW_FLOATS = (size_t)2 * (240 + TW_LIN + (SMEM_WM ? (SPLIT_WM ? 2 : 3) * (N / 2) : 0));
    // FSCAN_K4_GSTAGE_BODY (A/B, plain path below N = 1024): the CTA's G columns by
    // one TMA bulk copy into a stage behind the tables during the F pass
    static constexpr bool GST_BODY = FSCAN_K4_GSTAGE_BODY && N < 512;
    static constexpr size_t BODY_BASE = ((WORK_FLOATS + TW_FLOATS) * sizeof(float) + 127) / 128 * 128;
    static constexpr size_t SMEM = GST_BODY ? BODY_BASE + (size_t)COLS * N * sizeof(float2) : (WORK_FLOATS + TW_FLOATS) * sizeof(float);
    // explicit residency targets where ptxas' own choice leaves the SM
    // register-bound (N = 256: 4 CTAs of 192 threads; N = 1024: 3 of 192)
    // (N = 512 without the staged W_M table: 54 KB of shared memory, three CTAs
    // per SM at <= 96 registers: C4 +2% over the staged table at 80; four CTAs
    // at 80 registers run the kernel alone faster but the pipeline 1.5% slower)
    static constexpr int MIN_BLOCKS = N == 1024 ? 3 : (N == 256 ? 4 : (kK4W48 ? FSCAN_K4_MINB512 : 0));
    // inputs loaded and folded once per (column, n0) site for all three q and
    // parked in shared memory (N = 1024: C5 +3%); below, every q group loads and
    // folds its own elements (the shared fold measured 1% slower at N = 512)
    static constexpr bool FOLD1 = N >= 1024;
    static_assert(FOLD1 == !kFgtPlanes<N>, "K3 writes the layout this kernel reads");
    // merged-twiddle path (xlat_cols_merged, two-stage K-point transforms):
    // the exchange buffers + the [16][kQS] table W_M^{a j}
    static constexpr bool MERGE = kK4Merge && !FOLD1 && N == 512;
    // FSCAN_K4_GSTAGE (A/B): the CTA's G columns (COLS x N float2, contiguous in
    // the G plane) by one TMA bulk copy issued before the F pass, 1 = into their
    // own stage behind the table, 2 = into buffer B (idle until G's transform)
    // column blocks per pair, and per CTA on the merged path (FSCAN_K4_BLOCKS)
    static constexpr int NBLOCKS = (3 * N / 4 + 1 + COLS - 1) / COLS;
    static constexpr int NBLK = (kK4Merge && N == 512 && FSCAN_K4_GSTAGE == 1) ? FSCAN_K4_BLOCKS : 1;
    static constexpr size_t MERGE_BASE = ((FFT_FLOATS + 2 * 16 * fscan_fft::kQS) * sizeof(float) + 127) / 128 * 128;
    static constexpr size_t SMEM_MERGE = MERGE_BASE + (FSCAN_K4_GSTAGE == 1 ? (size_t)COLS * N * sizeof(float2) : 0);
};

template <int N>
__device__ __forceinline__ void xlat_cols_body(const Params& p);

template <int N>
__global__ void __launch_bounds__(XColGeom<N>::THREADS) k_xlat_cols(Params p) {
    xlat_cols_body<N>(p);
}

template <int N, int MINB>
__global__ void __launch_bounds__(XColGeom<N>::THREADS, MINB) k_xlat_cols_mb(Params p) {
    xlat_cols_body<N>(p);
}

// K4's two stores of combine slot j (m = q + 3 j, n0 = t + m T) go to rows
// half - n0 and half - n0 + K of the Y layout. When RB divides T, a row step of
// 3 T keeps the row's place inside its block, so both sequences are a base
// address minus compile-time multiples of 3 T / RB block strides.
template <int N>
struct YStores {
    static constexpr int RB = y_rows(N);
    float2* d0;
    float2* d1;
    __device__ __forceinline__ YStores(float2* dst, int t, int q, int T, int kp) {
        const int i0 = N / 2 - 1 - (t + q * T);
        d0 = dst + y_at<N>(i0, kp);
        d1 = dst + y_at<N>(i0 + N / 2, kp);
    }
    template <int T>
    __device__ __forceinline__ static constexpr int step(int j) {
        return -(3 * j * T / RB) * (3 * N / 4 + 1) * RB;
    }
};

template <int N>
__device__ __forceinline__ void xlat_cols_merged(const Params& p);

template <int N>
__device__ __forceinline__ void xlat_cols_body(const Params& p) {
    if constexpr (XColGeom<N>::MERGE) {
        xlat_cols_merged<N>(p);
        return;
    }
    constexpr int K = N / 2, M = 3 * K, H = M / 2;
    using X = XColGeom<N>;
    using G = typename X::G;
    constexpr int T = G::T, COLS = X::COLS;
    constexpr int half = N / 2 - 1;
    extern __shared__ __align__(128) float smem[];
    const int pair = blockIdx.y;
    int tr, t;
    G::map(threadIdx.x, tr, t);
    // (kK4QMajor, off: q-major transform order — a warp's two transforms one q
    // group of two adjacent columns — makes the radix-3 combine conflict-free
    // (bank model 162 -> 96 wavefronts) and q warp-uniform, but measured K4
    // 9.2 -> 9.6 ms and C2 -3%: the three q groups of a column no longer load
    // their shared fgt column from the same warp)
    constexpr bool QM = kK4QMajor && !X::FOLD1;
    const int c = QM ? tr % COLS : tr / 3, q = QM ? tr / COLS : tr % 3;
    const int kp = blockIdx.x * COLS + c;
    const int kq = kp <= H ? kp : H;  // the last block may hold fewer columns
    const auto bufA = G::lay(smem, tr);
    const auto bufB = G::lay(smem + G::FLOATS, tr);
    const float2* srcF = fgt_plane<N>(p, pair, 0) + (size_t)kq * N;
    const float2* srcG = fgt_plane<N>(p, pair, 1) + (size_t)kq * N;
    // stage the twiddle tables in shared memory (latency: the FFT stages and
    // input/combine twiddles read them ~90 times per thread)
    float2* stw_rk = reinterpret_cast<float2*>(smem + X::WORK_FLOATS);
    float2* stw_k = stw_rk + 240;
    float2* stw_m_s = stw_k + X::TW_LIN;
    // PF: every table load issued up front into registers and stored after the
    // first fold (a load -> store loop waits out one L2 round trip per trip)
    constexpr bool PF = !X::SMEM_WM;
    constexpr int TE = 240 + X::TW_LIN, TPT = PF ? (TE + X::THREADS - 1) / X::THREADS : 1;
    [[maybe_unused]] float2 tv[TPT];
    if constexpr (PF) {
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
            const int i = threadIdx.x + k * X::THREADS;
            if (TE % X::THREADS == 0 || i < TE) tv[k] = __ldg(i < 240 ? p.tw_rk + i : p.tw_k + (i - 240));
        }
    } else {
        for (int i = threadIdx.x; i < 240; i += X::THREADS) stw_rk[i] = __ldg(p.tw_rk + i);
        for (int i = threadIdx.x; i < X::TW_LIN; i += X::THREADS) stw_k[i] = __ldg(p.tw_k + i);
    }
    auto tw_store = [&]() {  // stw_k follows stw_rk
        if constexpr (PF) {
#pragma unroll
            for (int k = 0; k < TPT; ++k) {
                const int i = threadIdx.x + k * X::THREADS;
                if (TE % X::THREADS == 0 || i < TE) stw_rk[i] = tv[k];
            }
        }
    };
    if constexpr (X::SMEM_WM && X::SPLIT_WM) {
        for (int i = threadIdx.x; i < K; i += X::THREADS) {
            stw_m_s[i] = __ldg(p.tw_m + i);
            stw_m_s[K + i] = __ldg(p.tw_m + 2 * i);
        }
    } else if constexpr (X::SMEM_WM) {
        for (int i = threadIdx.x; i < M; i += X::THREADS) stw_m_s[i] = __ldg(p.tw_m + i);
    }
    auto wq = [&](int n0, int qq) {
        if constexpr (X::SMEM_WM && X::SPLIT_WM) return stw_m_s[(qq - 1) * K + n0];
        else if constexpr (X::SMEM_WM) return stw_m_s[qq * n0];
        else return __ldg(p.tw_m + qq * n0);
    };
    // kK4W48: the thread's twiddle bases (see the W_48 table above)
    const float2 bq = X::FOLD1 ? make_float2(1.f, 0.f) : __ldg(p.tw_m + q * t);  // W_M^{q t}
    const float2 b1 = (X::FOLD1 && !kK4W48Fold1) ? make_float2(1.f, 0.f) : __ldg(p.tw_m + t);      // W_M^{t}
    const float2 b2 = (X::FOLD1 && !kK4W48Fold1) ? make_float2(1.f, 0.f) : __ldg(p.tw_m + 2 * t);  // W_M^{2 t}
    auto wq_m = [&](int m, int n0) {  // W_M^{q n0}, n0 = t + m T
        if constexpr (kK4W48 && !X::FOLD1) return cmul(bq, w48(q * m));
        else return wq(n0, q);
    };
    pdl_enter();
    [[maybe_unused]] __shared__ uint64_t g_bar;
    [[maybe_unused]] float2* gst = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem) + X::BODY_BASE);
    if constexpr (X::GST_BODY) {
        if (threadIdx.x == 0) {
            const int k0 = blockIdx.x * COLS;
            const int nc = (H + 1 - k0) < COLS ? (H + 1 - k0) : COLS;
            mbar_init(&g_bar, 1);
            bulk_load(gst, fgt_plane<N>(p, pair, 1) + (size_t)k0 * N, (unsigned)(nc * N * sizeof(float2)), &g_bar);
        }
    }
    // LATE: the F fold reads no staged table, so its global loads are issued
    // before the barrier that publishes the twiddle tables (the table and input
    // load latencies overlap instead of following one another)
    constexpr bool LATE = kK4LateSync && !X::FOLD1 && !X::SMEM_WM;
    if constexpr (!LATE && !X::FOLD1) {
        tw_store();
        __syncthreads();
    }
#ifdef FSCAN_K4_TWPOW
    const float2* twk = p.tw_k;  // A/B: powers of four global-table reads (fft.cuh kTwPow)
#else
    const fscan_fft::SmemTwRK twk{stw_rk, stw_k};
#endif
    const float2 w3q = w3(q);
    float2 a[16];
    if constexpr (X::FOLD1) {
        // one thread per (column, n0): (F, G) at n0 and n0 + K loaded once, the
        // three q inputs of both transforms formed together (a radix-3 butterfly
        // with x2 = 0) and parked in the transforms' exchange buffers (F in A, G
        // in B); the q groups then read their inputs from shared memory (instead
        // of each loading and folding every element itself: 3x fewer global loads)
        constexpr int SITES = COLS * K, ITER = (SITES + X::THREADS - 1) / X::THREADS;
        [[maybe_unused]] const float2 fb1 = kK4Fold1Base ? __ldg(p.tw_m + threadIdx.x) : make_float2(1.f, 0.f);
        float4 v0[ITER], v1[ITER];  // every load in flight before the first use
#pragma unroll
        for (int it = 0; it < ITER; ++it) {
            const int e = threadIdx.x + it * X::THREADS;
            if (SITES % X::THREADS == 0 || e < SITES) {
                const int cc = e / K, n0 = e % K;
                const int kc = min((int)blockIdx.x * COLS + cc, H);
                static_assert(!kFgtPlanes<N>, "FOLD1 reads the interleaved (F, G) layout");
                const float4* s4 = reinterpret_cast<const float4*>(p.fgt) + ((size_t)pair * (H + 1) + kc) * N;
                v0[it] = s4[n0];
                v1[it] = s4[n0 + K];
            }
        }
#pragma unroll
        for (int it = 0; it < ITER; ++it) {
            const int e = threadIdx.x + it * X::THREADS;
            if (!(SITES % X::THREADS == 0 || e < SITES)) break;
            const int cc = e / K, n0 = e % K;
            const float4 u0 = v0[it], u1 = v1[it];
            float2 w1, w2;  // W_M^{n0}, W_M^{2 n0}
            if constexpr (kK4Fold1Base && M == 8 * X::THREADS) {
                // n0 = e - cc K with e = tid + it THREADS: W_M^{n0} = W_M^{tid}
                // W_8^{it} W_3^{-cc} (M = 8 THREADS; W_M^K = W_3): the thread's one
                // table read times constants instead of two table reads per site
                float2 w = it == 0 ? fb1 : cmul(fb1, fscan_fft::w16c<-1>(2 * it));
                if (cc) w = cmul(w, make_float2(-0.5f, kS3));
                w1 = w;
                w2 = cmul(w, w);
            } else {
                w1 = wq(n0, 1);
                w2 = wq(n0, 2);
            }
            auto fold = [&](float2 x0, float2 x1, float* base) {
                const float2 tt = make_float2(fmaf(-0.5f, x1.x, x0.x), fmaf(-0.5f, x1.y, x0.y));
                const float2 ss = make_float2(kS3 * x1.x, kS3 * x1.y);
                G::lay(base, 3 * cc).put(n0, cadd(x0, x1));
                G::lay(base, 3 * cc + 1).put(n0, cmul(w1, make_float2(tt.x + ss.y, tt.y - ss.x)));
                G::lay(base, 3 * cc + 2).put(n0, cmul(w2, make_float2(tt.x - ss.y, tt.y + ss.x)));
            };
            fold(make_float2(u0.x, u0.y), make_float2(u1.x, u1.y), smem);
            fold(make_float2(u0.z, u0.w), make_float2(u1.z, u1.w), smem + G::FLOATS);
        }
        tw_store();
        __syncthreads();  // the folded inputs and the tables
#pragma unroll
        for (int m = 0; m < 16; ++m) a[m] = bufA.get(t + m * T);
        __syncwarp();  // every input read before the transform's exchange writes
    } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int n0 = t + m * T;
            const float2 s = cadd(srcF[n0], cmul(w3q, srcF[n0 + K]));
            a[m] = q ? cmul(wq_m(m, n0), s) : s;
        }
        if constexpr (LATE) {
            tw_store();
            __syncthreads();
        }
    }
    fft_regs<K, -1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufA, twk);  // transforms of a warp share a buffer group
#pragma unroll
    for (int m = 0; m < 16; ++m) bufA.put(t + m * T, a[m]);  // park F_q (own slots)
    if constexpr (X::FOLD1) {
#pragma unroll
        for (int m = 0; m < 16; ++m) a[m] = bufB.get(t + m * T);
        __syncwarp();
    } else {
        const float2* gs = srcG;
        if constexpr (X::GST_BODY) {
            static_assert(!X::GST_BODY || (kK4LateSync && !X::SMEM_WM), "the table barrier publishes g_bar");
            mbar_wait(&g_bar, 0);
            gs = gst + (kq - blockIdx.x * COLS) * N;
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int n0 = t + m * T;
            const float2 s = cadd(gs[n0], cmul(w3q, gs[n0 + K]));
            a[m] = q ? cmul(wq_m(m, n0), s) : s;
        }
    }
    fft_regs<K, -1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufB, twk);
#pragma unroll
    for (int m = 0; m < 16; ++m) a[m] = cmul(cconj(bufA.get(t + m * T)), a[m]);  // conj(F) G
    if (p.phase) {  // opt-in phase correlation: X / |X| (0 where X = 0), SURVEY a21
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const float mag = sqrtf(a[m].x * a[m].x + a[m].y * a[m].y);
            const float inv = mag > 0.0f ? 1.0f / mag : 0.0f;
            a[m] = make_float2(a[m].x * inv, a[m].y * inv);
        }
    }
    fft_regs<K, +1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufB, twk);
#pragma unroll
    for (int m = 0; m < 16; ++m) bufB.put(t + m * T, a[m]);
    __syncthreads();
    // radix-3 combine: group q handles the slots m = q, q+3, ... of its column
    auto tr_of = [&](int qq) { return QM ? qq * COLS + c : 3 * c + qq; };
    const auto e0 = G::lay(smem + G::FLOATS, tr_of(0)), e1 = G::lay(smem + G::FLOATS, tr_of(1)),
               e2 = G::lay(smem + G::FLOATS, tr_of(2));
    const float2 w31 = w3(1), w32 = w3(2);
    // outputs straight into K5's row blocks (y_at; stored by surface row
    // i = half - ky, the flip of matcher.cpp:171-182): the 16 lanes of a
    // transform hold 16 consecutive rows of one bin, whole RB-row runs
    float2* dst = p.zbuf + (size_t)pair * N * (H + 1);
    const bool store = kp <= H;  // the last block's clamped duplicates store nothing
    [[maybe_unused]] const YStores<N> ys(dst, t, q, T, kp);
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        const int m = q + 3 * j;
        if (m < 16) {
            const int n0 = t + m * T;
            float2 v1, v2;  // W_M^{n0}, W_M^{2 n0}
            if constexpr (kK4W48 && (!X::FOLD1 || kK4W48Fold1)) {
                v1 = cmul(b1, w48(m));
                v2 = cmul(b2, w48(2 * m));
            } else {
                v1 = wq(n0, 1);
                v2 = wq(n0, 2);
            }
            const float2 x0 = e0.get(n0);
            const float2 x1 = cmul(cconj(v1), e1.get(n0));
            const float2 x2 = cmul(cconj(v2), e2.get(n0));
            if (store) {
                const float2 o0 = cadd(x0, cadd(x1, x2)), o1 = cadd(x0, cadd(cmul(w31, x1), cmul(w32, x2)));
                if constexpr (T % YStores<N>::RB == 0) {
                    ys.d0[YStores<N>::template step<T>(j)] = o0;
                    ys.d1[YStores<N>::template step<T>(j)] = o1;
                } else {
                    dst[y_at<N>(half - n0, kp)] = o0;
                    dst[y_at<N>(half - (n0 - K), kp)] = o1;
                }
            }
        }
    }
}

// K4 with merged twiddles (N <= 512): the same transforms and combine as
// xlat_cols_body, with every W_M factor either folded into the last FFT stage's
// twiddles (fft.cuh SmemTwQF / SmemTwQI) or applied once per value:
//   F_q: inputs W_M^{mTq} (x[n] + W_3^q x[n+K]), last stage F[r][3k+q];
//   e_q: last stage conj(F[k][3r+q]), outputs W_M^{-16 r' q} — so e_q arrives
//        pre-multiplied by the combine twiddle W_M^{-n q};
//   combine: sum_q x_q and x_0 - (x_1 + x_2)/2 - i (sqrt 3/2)(x_1 - x_2).
// The fold W_3^q product is two FMAs per component with per-thread constants.
template <int N>
__device__ __forceinline__ void xlat_cols_merged(const Params& p) {
    constexpr int K = N / 2, H = 3 * K / 2;
    using X = XColGeom<N>;
    using G = typename X::G;
    constexpr int T = G::T, COLS = X::COLS;
    constexpr int R = K / 16, NB = 16 / R;  // last-stage radix and butterflies per thread
    [[maybe_unused]] constexpr int QS = fscan_fft::kQS;
    constexpr int half = N / 2 - 1;
    static_assert(K >= 32 && K <= 256 && R * 16 == K, "two-stage K-point transforms");
    extern __shared__ __align__(128) float smem[];
    const int pair = blockIdx.y;
    int tr, t;
    G::map(threadIdx.x, tr, t);
    const int c = tr / 3, q = tr % 3;
    // NBLK consecutive column blocks per CTA (X::NBLK > 1 needs the G stage): the
    // first block's F columns come by per-thread loads, every later block's by a
    // bulk copy into the stage issued while the block before it is still in its
    // product / inverse / combine phases; the stage alternates G(b), F(b+1),
    // G(b+1), ... (`e_bar` counts the threads done reading it)
    constexpr int GST = FSCAN_K4_GSTAGE;
    constexpr int NBLK = X::NBLK;
    static_assert(NBLK == 1 || GST == 1, "several blocks per CTA stream through the G stage");
    const int b0 = blockIdx.x * NBLK;
    const int nb = NBLK == 1 ? 1 : (X::NBLOCKS - b0 < NBLK ? X::NBLOCKS - b0 : NBLK);
    const auto bufA = G::lay(smem, tr);
    const auto bufB = G::lay(smem + G::FLOATS, tr);
    float2* tab = reinterpret_cast<float2*>(smem + X::FFT_FLOATS);  // [16][QS]
    // the table's global loads are all issued first and stored to shared memory
    // only after the first fold (a load -> store loop waited out one L2 round
    // trip per iteration: ~15% of K4's warp samples)
    // (kK4TabGlobal: the stages read the table through L1 from global memory —
    // no per-CTA staging, its loads or its barrier)
    constexpr int TE = 16 * 48, TPT = kK4TabGlobal ? 1 : (TE + X::THREADS - 1) / X::THREADS;
    [[maybe_unused]] float2 tv[TPT];
    if constexpr (!kK4TabGlobal) {
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
            const int i = threadIdx.x + k * X::THREADS;
            if (TE % X::THREADS == 0 || i < TE) tv[k] = __ldg(p.tw_k4 + i);
        }
    }
    pdl_enter();
    [[maybe_unused]] __shared__ uint64_t g_bar, f_bar, e_bar, t_bar;
    [[maybe_unused]] float2* gst = reinterpret_cast<float2*>(
        GST == 1 ? reinterpret_cast<char*>(smem) + X::MERGE_BASE : reinterpret_cast<char*>(smem + G::FLOATS));
    // the stage <- the (up to) COLS columns of block `blk` of plane 0 (F) / 1 (G)
    [[maybe_unused]] auto stage_block = [&](int plane, int blk, uint64_t* bar) {
        const int k0 = blk * COLS;
        const int nc = (H + 1 - k0) < COLS ? (H + 1 - k0) : COLS;
        bulk_load(gst, fgt_plane<N>(p, pair, plane) + (size_t)k0 * N, (unsigned)(nc * N * sizeof(float2)), bar);
    };
    // kK4SplitTab: the table's barrier split into an arrive (after a thread's
    // table stores) and a wait just before the first transform's last stage
    // (fft.cuh TwQF<.., W>), so no warp waits out the slowest warp's F loads
    // before its first FFT stage
    constexpr bool SPLIT = kK4SplitTab && GST != 0 && !kK4TabGlobal;
    if constexpr (GST != 0) {
        static_assert(GST == 1 || G::FLOATS * sizeof(float) >= (size_t)COLS * N * sizeof(float2), "buffer B holds the G columns");
        if (threadIdx.x == 0) {
            mbar_init(&g_bar, 1);
            if constexpr (SPLIT) mbar_init(&t_bar, X::THREADS);
            if constexpr (NBLK > 1) {
                mbar_init(&f_bar, 1);
                mbar_init(&e_bar, X::THREADS);
            }
            stage_block(1, b0, &g_bar);
        }
        if constexpr (SPLIT) __syncthreads();  // publishes the mbarriers (no warp has a load in flight yet)
    }
    // W_3^q = (c1, wi): s = x0 + W_3^q x1 in four FMAs
    const float c1 = q ? -0.5f : 1.0f, wi = q == 0 ? 0.0f : (q == 1 ? -kS3 : kS3);
    const float2* fq = kK4TabGlobal ? p.tw_k4 + q : tab + q;  // F[.][3k + q]
    using TQF = std::conditional_t<kK4TabGlobal, fscan_fft::TwQF<48, true>, fscan_fft::SmemTwQF>;
    using TQI = std::conditional_t<kK4TabGlobal, fscan_fft::TwQI<48, true>, fscan_fft::SmemTwQI>;
    // W_M^{m T q} = W_48^{m q} and W_M^{16 r' q} = W_48^{(16 / R) r' q} from the
    // constant-bank table (one address per half-warp)
    auto win = [&](int m) { return w48(m * q); };
    auto wout = [&](int r) { return w48((16 / R) * r * q); };
    auto fold = [&](float2 x0, float2 x1, int m) {
        const float2 sv = make_float2(fmaf(-wi, x1.y, fmaf(c1, x1.x, x0.x)), fmaf(wi, x1.x, fmaf(c1, x1.y, x0.y)));
        return cmul(sv, win(m));
    };
    float2* dst = p.zbuf + (size_t)pair * N * (H + 1);
    [[maybe_unused]] unsigned ephase = 0;
#pragma unroll 1
    for (int ib = 0; ib < nb; ++ib) {
        const int blk = b0 + ib;
        const int kp = blk * COLS + c;
        const int kq = kp <= H ? kp : H;  // the last block may hold fewer columns
        [[maybe_unused]] const float2* stg = gst + (kq - blk * COLS) * N;  // this thread's column in the stage
        float2 a[16];
        if (NBLK == 1 || ib == 0) {
            const float2* srcF = fgt_plane<N>(p, pair, 0) + (size_t)kq * N;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int n0 = t + m * T;
                a[m] = fold(srcF[n0], srcF[n0 + K], m);
            }
            if constexpr (!kK4TabGlobal) {
#pragma unroll
                for (int k = 0; k < TPT; ++k) {
                    const int i = threadIdx.x + k * X::THREADS;
                    if (TE % X::THREADS == 0 || i < TE) tab[(i / 48) * QS + i % 48] = tv[k];
                }
                if constexpr (SPLIT)
                    mbar_arrive(&t_bar);
                else
                    __syncthreads();  // the table (the fold reads none of it) and the mbarriers
            }
        } else {
            mbar_wait(&f_bar, (ib - 1) & 1);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int n0 = t + m * T;
                a[m] = fold(stg[n0], stg[n0 + K], m);
            }
            mbar_arrive(&e_bar);
            if (threadIdx.x == 0) {  // every thread has read F: the stage takes this block's G
                mbar_wait(&e_bar, ephase);
                stage_block(1, blk, &g_bar);
            }
            ephase ^= 1;
        }
        if constexpr (SPLIT)
            fft_regs<K, -1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufA, fscan_fft::TwQF<fscan_fft::kQS, false, true>{fq, &t_bar});
        else
            fft_regs<K, -1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufA, TQF{fq});
#pragma unroll
        for (int m = 0; m < 16; ++m) bufA.put(t + m * T, a[m]);  // park F_q (own slots)
        if constexpr (GST != 0) {
            static_assert(!kK4TabGlobal, "the table barrier publishes g_bar");
            mbar_wait(&g_bar, ib & 1);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int n0 = t + m * T;
                a[m] = fold(stg[n0], stg[n0 + K], m);
            }
            if constexpr (GST == 2) __syncthreads();  // every staged read before buffer B's exchange writes
            if constexpr (NBLK > 1) {
                if (ib + 1 < nb) {
                    mbar_arrive(&e_bar);
                    if (threadIdx.x == 0) {  // every thread has read G: the stage takes the next block's F
                        mbar_wait(&e_bar, ephase);
                        stage_block(0, blk + 1, &f_bar);
                    }
                    ephase ^= 1;
                }
            }
        } else {
            const float2* srcG = fgt_plane<N>(p, pair, 1) + (size_t)kq * N;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int n0 = t + m * T;
                a[m] = fold(srcG[n0], srcG[n0 + K], m);
            }
        }
        fft_regs<K, -1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufB, TQF{fq});
#pragma unroll
        for (int m = 0; m < 16; ++m) a[m] = cmul(cconj(bufA.get(t + m * T)), a[m]);  // conj(F) G
        if (p.phase) {  // opt-in phase correlation: X / |X| (0 where X = 0), SURVEY a21
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const float mag = sqrtf(a[m].x * a[m].x + a[m].y * a[m].y);
                const float inv = mag > 0.0f ? 1.0f / mag : 0.0f;
                a[m] = make_float2(a[m].x * inv, a[m].y * inv);
            }
        }
        fft_regs<K, +1, true, (kPk<N> ? FSCAN_PK_K4 : 0)>(a, t, bufB, TQI{fq});
#pragma unroll
        for (int m = 0; m < 16; ++m) bufB.put(t + m * T, cmul(a[m], cconj(wout(m / NB))));
        // the combine of column c reads the three transforms 3c .. 3c + 2: with
        // COLS = 4 and 16 threads per transform, columns (0, 1) live in warps 0-2
        // and (2, 3) in warps 3-5, so a 96-thread named barrier per column pair
        // is enough (kK4PairBar, A/B)
        if constexpr (kK4PairBar && NBLK == 1 && COLS == 4 && T == 16 && X::THREADS == 192)
            asm volatile("bar.sync %0, 96;" ::"r"(1 + (int)(threadIdx.x >= 96)) : "memory");
        else
            __syncthreads();
        // radix-3 combine of the pre-twiddled e_q; group q handles slots m = q, q+3, ...
        // (several blocks per CTA: the next block's first write to buffer B follows
        // its wait on g_bar, i.e. every thread's arrival after this combine)
        const auto e0 = G::lay(smem + G::FLOATS, 3 * c), e1 = G::lay(smem + G::FLOATS, 3 * c + 1),
                   e2 = G::lay(smem + G::FLOATS, 3 * c + 2);
        const bool store = kp <= H;
        [[maybe_unused]] const YStores<N> ys(dst, t, q, T, kp);
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const int m = q + 3 * j;
            if (m < 16) {
                const int n0 = t + m * T;
                const float2 x0 = e0.get(n0), x1 = e1.get(n0), x2 = e2.get(n0);
                const float2 sa = cadd(x1, x2), df = csub(x1, x2);
                if (store) {
                    const float2 o0 = cadd(x0, sa);
                    const float2 o1 = make_float2(fmaf(kS3, df.y, fmaf(-0.5f, sa.x, x0.x)),
                                                  fmaf(-kS3, df.x, fmaf(-0.5f, sa.y, x0.y)));
                    if constexpr (T % YStores<N>::RB == 0) {
                        ys.d0[YStores<N>::template step<T>(j)] = o0;
                        ys.d1[YStores<N>::template step<T>(j)] = o1;
                    } else {
                        dst[y_at<N>(half - n0, kp)] = o0;
                        dst[y_at<N>(half - (n0 - K), kp)] = o1;
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------- K5
// Surface row i: real inverse of length M along x from the Hermitian half
// Y[0..M/2] as one complex inverse of length M/2 = 3 K2 (K2 = K/2):
//   A[k] = Y[k] + conj Y[M/2-k], B[k] = (Y[k] - conj Y[M/2-k]) W_M^{-k},
//   z = IFFT_{M/2}(A + iB) = sum_q W_M^{-2nq} W_3^{-sq} IFFT_K2(Z_q)[n0], n = n0 + s K2,
//   x[2n] = Re z[n], x[2n+1] = Im z[n];
// group q inverts Z_q; scaled by 1/M^2, cropped to lags kx in [-(N/2-1), N/2]
// (surface col j = kx + half), plus this block's hard argmax (lowest index on ties).
#ifdef FSCAN_K5_ROWMAJOR
constexpr bool kK5QMajor = false;  // A/B: transforms ordered row-major (3 rl + q)
#else
constexpr bool kK5QMajor = true;
#endif
#ifdef FSCAN_K5_TW_TABLE
constexpr bool kK5TwTable = true;  // A/B: input / combine twiddles read from the W_M table per element
#else
constexpr bool kK5TwTable = false;
#endif
#ifdef FSCAN_K5_LDG
constexpr bool kK5Tma = false;  // A/B: every thread loads its Y elements from global
#else
constexpr bool kK5Tma = true;
#endif

template <int N>
struct XOutGeom {
    static constexpr int K2 = N / 4;
    static constexpr int T = K2 / 16;
    // 192 threads (3 transforms per row): N = 512 runs K5 7% faster than at 384
    // (more, shorter CTAs per SM); the doubled block maxima cost K6 nothing
    // since warp 0 reduces them in parallel
    static constexpr int ROWS0 = 64 / T;
    static constexpr int ROWS = ROWS0 < N ? ROWS0 : N;
    static constexpr int THREADS = 3 * ROWS * T;
    using G = Geom<K2, THREADS>;
    static_assert(ROWS == y_rows(N), "one K5 CTA inverts one block of the Y layout");
    // the CTA's block of Y (ROWS rows, [k'][ROWS] contiguous, y_at) arrives by one
    // TMA bulk copy into the same shared memory the FFT exchange uses afterwards
    static constexpr size_t YBYTES = (size_t)ROWS * (3 * N / 4 + 1) * sizeof(float2);
    static constexpr size_t FFT_BYTES = (size_t)G::FLOATS * sizeof(float);
    static constexpr size_t SMEM = (kK5Tma && YBYTES > FFT_BYTES) ? YBYTES : FFT_BYTES;
};

// EMB: only the lag window [win_off, win_off + p.n)^2 of the embedded surface
// competes for the argmax, and the surface stays in the workspace (K6 copies
// the window out).
// MODE (kOutFull / kOutMax / kOutWin): the full surface (rows stored unless
// p.skip_surface), or the two-pass throughput form — kOutMax keeps only the
// block maxima (no surface store: 4N^2 bytes and ~20 STG per thread less),
// then kOutWin recomputes just the row blocks the soft-argmax window of the
// pair's peak touches (grid.x = window blocks, the peak reduced from the
// kOutMax partials exactly as K6 reduces them) and stores those rows; the
// values are the same instructions on the same inputs, so bit-identical.
constexpr int kOutFull = 0, kOutMax = 1, kOutWin = 2;

__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
    if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
    }
}

#ifdef FSCAN_K5_MINB
#define FSCAN_K5_BOUNDS __launch_bounds__(XOutGeom<N>::THREADS, FSCAN_K5_MINB)
#else
#define FSCAN_K5_BOUNDS __launch_bounds__(XOutGeom<N>::THREADS)
#endif
template <int N, bool EMB, int MODE = kOutFull>
__global__ void FSCAN_K5_BOUNDS k_xlat_out(Params p) {
    pdl_enter();
    constexpr int K = N / 2, M = 3 * K, H = M / 2;
    using X = XOutGeom<N>;
    using G = typename X::G;
    constexpr int THREADS = X::THREADS, ROWS = X::ROWS;
    constexpr int NW = THREADS / 32;
    constexpr int T = G::T;
    constexpr int half = N / 2 - 1;
    extern __shared__ __align__(128) float smem[];
    __shared__ float red_v[NW];
    __shared__ int red_i[NW];
    const int pair = blockIdx.y;
    int blk = blockIdx.x;
    __shared__ int win_blk, win_r0, win_r1, win_c0, win_c1;  // kOutWin: the peak's window
    if constexpr (MODE == kOutWin) {
        // the pair's peak from the kOutMax block maxima (K6's reduction), then
        // this CTA's block among those rows [pr - w, pr + w] touches
        if (threadIdx.x < 32) {
            constexpr int NP = N / ROWS;
            const Partial* pp = p.part + (size_t)pair * NP;
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int b = threadIdx.x; b < NP; b += 32) better(bv, bi, pp[b].val, pp[b].idx);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                better(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
            if (threadIdx.x == 0) {
                const int pk = bi == 0x7fffffff ? 0 : bi, pr = pk / N, pc = pk % N;
                win_r0 = max(0, pr - p.window);
                win_r1 = min(N - 1, pr + p.window);
                win_c0 = max(0, pc - p.window);
                win_c1 = min(N - 1, pc + p.window);
                const int b0 = win_r0 / ROWS, b1 = win_r1 / ROWS;
                win_blk = b0 + (int)blockIdx.x <= b1 ? b0 + (int)blockIdx.x : -1;
            }
        }
        __syncthreads();
        blk = win_blk;
        if (blk < 0) return;
    }
    int tr, t;
    G::map(threadIdx.x, tr, t);
    // q-major transform order (kK5QMajor): the transforms of a half-warp are one
    // q group of adjacent rows; with the row permutation of the Y blocks their
    // stride-3 bin reads fall on distinct bank pairs (y_swz)
    const int rl = kK5QMajor ? tr % ROWS : tr / 3, q = kK5QMajor ? tr / ROWS : tr % 3;
    const int i = blk * ROWS + rl;
    const auto buf = G::lay(smem, tr);
    {
        // kK5Tma: the block by one bulk copy (the per-thread global loads of the
        // stride-3 pattern left every warp waiting on its own loads; a per-thread
        // cp.async staging measured slower than those loads)
        const float2* yblk = p.zbuf + ((size_t)pair * N + blk * ROWS) * (H + 1);
        if constexpr (kK5Tma) {
            __shared__ uint64_t mbar;
            if (threadIdx.x == 0) mbar_init(&mbar, 1);
            __syncthreads();
            if (threadIdx.x == 0) bulk_load(smem, yblk, (unsigned)X::YBYTES, &mbar);
            mbar_wait(&mbar, 0);
            yblk = reinterpret_cast<const float2*>(smem);
        }
        auto y = [&](int k) { return yblk[k * ROWS + (rl ^ y_swz(ROWS, k))]; };  // Y[i][k]
        // W_M^k, k = 3 (t + m T) + q (M = 96 T): the thread's base W_M^{3t+q}
        // times W_32^m, a compile-time constant-bank address (kK5TwTable: one
        // scattered W_M table read per element, ~40% of K5's L1 wavefronts)
        const float2 bk = kK5TwTable ? make_float2(1.f, 0.f) : wm(p.tw_m, 3 * t + q);
        // the bins k0 + 3 T m (and H - k0 - 3 T m) of this thread keep the row
        // permutation of k0 whenever 3 T is a multiple of y_swz's bit period (N >= 256):
        // one base address per direction, compile-time offsets 3 T m RB
        constexpr int SWB = ROWS >= 16 ? 0 : (ROWS == 8 ? 1 : 2);
        constexpr bool HOIST = (3 * T) % (4 << SWB) == 0;
        const int k0 = 3 * t + q;
        const float2* yf = yblk + k0 * ROWS + (rl ^ y_swz(ROWS, k0));
        const float2* yb = yblk + (H - k0) * ROWS + (rl ^ y_swz(ROWS, H - k0));
        float2 v[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int k = 3 * (t + m * T) + q;
            const float2 a = HOIST ? yf[3 * T * m * ROWS] : y(k);
            const float2 b = cconj(HOIST ? yb[-3 * T * m * ROWS] : y(H - k));
            const float2 A = cadd(a, b);
            const float2 wk = kK5TwTable ? wm(p.tw_m, k) : cmul(bk, w32(m));
            const float2 B = cmul(csub(a, b), cconj(wk));
            v[m] = make_float2(A.x - B.y, A.y + B.x);  // A + iB
        }
        if constexpr (kK5Tma) __syncthreads();  // Y reads done before the exchange reuses the bytes
        fft_regs<X::K2, +1, true, (kPk<N> ? FSCAN_PK_K5 : 0)>(v, t, buf, p.tw_k2);
#pragma unroll
        for (int m = 0; m < 16; ++m) buf.put(t + m * T, v[m]);
    }
    __syncthreads();
    const float scale = 1.0f / ((float)M * (float)M);
    float* srow = ((p.xy_surf && !EMB) ? p.xy_surf : p.surf) + ((size_t)pair * N + i) * N;
    const bool row_in = !EMB || (i >= p.win_off && i < p.win_off + p.n);
    bool win_row = false;
    if constexpr (MODE == kOutWin) win_row = i >= win_r0 && i <= win_r1;
    float best_v = -INFINITY;
    int best_i = 0x7fffffff;
    auto emit = [&](int kx, float val) {
        const int j = kx + half;
        if constexpr (MODE == kOutWin) {  // only the window cells K6 reads
            if (win_row && j >= win_c0 && j <= win_c1) srow[j] = val;
            return;
        }
        if (MODE == kOutFull && !p.skip_surface) srow[j] = val;
        const int li = i * N + j;
        if (EMB && !(row_in && j >= p.win_off && j < p.win_off + p.n)) return;
        if (val > best_v || (val == best_v && li < best_i)) {
            best_v = val;
            best_i = li;
        }
    };
    auto tr_of = [&](int qq) { return kK5QMajor ? qq * ROWS + rl : 3 * rl + qq; };
    const auto e0 = G::lay(smem, tr_of(0)), e1 = G::lay(smem, tr_of(1)), e2 = G::lay(smem, tr_of(2));
    const float2 w31 = w3(1), w32 = w3(2);
    // W_M^{2 n0} = W_M^{2t} W_48^m and W_M^{4 n0} = W_M^{4t} W_48^{2m} (n0 = t + m T)
    const float2 b2 = kK5TwTable ? make_float2(1.f, 0.f) : wm(p.tw_m, 2 * t);
    const float2 b4 = kK5TwTable ? make_float2(1.f, 0.f) : wm(p.tw_m, 4 * t);
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        const int m = q + 3 * j;
        if (m < 16) {
            const int n0 = t + m * T;
            const float2 x0 = e0.get(n0);
            const float2 v2 = kK5TwTable ? wm(p.tw_m, 2 * n0) : cmul(b2, w48(m));
            const float2 v4 = kK5TwTable ? wm(p.tw_m, 4 * n0) : cmul(b4, w48(2 * m));
            const float2 x1 = cmul(cconj(v2), e1.get(n0));
            const float2 x2 = cmul(cconj(v4), e2.get(n0));
            const float2 z0 = cadd(x0, cadd(x1, x2));                        // s = 0
            const float2 z2 = cadd(x0, cadd(cmul(w31, x1), cmul(w32, x2)));  // s = 2: W_3^{-2q} = W_3^{q}
            emit(2 * n0, z0.x * scale);                   // pos 2n0, 2n0+1 -> kx = pos
            emit(2 * n0 + 1, z0.y * scale);
            if (n0 >= 1) emit(2 * n0 - K, z2.x * scale);  // pos 2n0+2K -> kx = 2n0-K
            emit(2 * n0 + 1 - K, z2.y * scale);
            if (n0 == 0) {  // s = 1, n0 = 0: pos K -> kx = N/2
                const float2 z1 = cadd(x0, cadd(cmul(cconj(w31), x1), cmul(cconj(w32), x2)));  // W_3^{-q}
                emit(K, z1.x * scale);
            }
        }
    }
    if constexpr (MODE != kOutWin) {  // block maximum -> p.part
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
            for (int w = 1; w < NW; ++w)
                if (red_v[w] > best_v || (red_v[w] == best_v && red_i[w] < best_i)) {
                    best_v = red_v[w];
                    best_i = red_i[w];
                }
            p.part[(size_t)pair * gridDim.x + blk] = Partial{best_v, best_i};
        }
    }
}

// ---------------------------------------------------------------- K6
constexpr int kFinThreads = 256;

// three sums in one pass (one pair of barriers instead of three); every value is
// reduced in the same order as block_sum
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    constexpr int NW = kFinThreads / 32;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x >> 5] = a;
        sh[NW + (threadIdx.x >> 5)] = b;
        sh[2 * NW + (threadIdx.x >> 5)] = c;
    }
    __syncthreads();
    a = b = c = 0.0;
    for (int w = 0; w < NW; ++w) {
        a += sh[w];
        b += sh[NW + w];
        c += sh[2 * NW + w];
    }
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
    pdl_enter();
    __shared__ double sh[kFinThreads / 32];
    __shared__ double sh3[3 * (kFinThreads / 32)];
    __shared__ float pk_v;
    __shared__ int pk_i;
    __shared__ double pre_sn, pre_cs, pre_th;
    const int pair = blockIdx.x;
    const int n = p.np;
    if (threadIdx.x == 32) {
        // the rotation's sine / cosine and normalised angle, computed by warp 1
        // while warp 0 reduces the block maxima (off thread 0's serial tail)
        const double theta = p.rot[pair].theta;
        double sn, cs;
        sincos(theta, &sn, &cs);  // rotate_vec (geometry.cpp:31-35)
        const double two_pi = 6.283185307179586;
        const double pi = 3.141592653589793;
        double th = fmod(theta, two_pi);  // normalize_angle (geometry.cpp:9-14)
        if (th <= -pi) th += two_pi;
        if (th > pi) th -= two_pi;
        pre_sn = sn;
        pre_cs = cs;
        pre_th = th;
    }
    if (threadIdx.x < 32) {
        // the K5 block maxima reduced by warp 0: the largest value, the lowest
        // linear index among equal values (an order-independent maximum, so the
        // same cell as the reference's strict-> row-major scan)
        const Partial* pp = p.part + (size_t)pair * nparts;
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int b = threadIdx.x; b < nparts; b += 32) {
            const Partial c = pp[b];
            if (c.val > bv || (c.val == bv && c.idx < bi)) {
                bv = c.val;
                bi = c.idx;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        // no ordered maximum (an all-NaN surface): the reference's strict-> scan
        // keeps its first cell, the window's (0, 0)
        if (threadIdx.x == 0) {
            const int o0 = p.embed ? p.win_off : 0;
            pk_v = bv;
            pk_i = bi == 0x7fffffff ? o0 * n + o0 : bi;
        }
    }
    __syncthreads();
    // the surface is n x n (pitch n = np); embedded grids keep
    // the reference's window of nv x nv lags at offset off
    const int nv = p.embed ? p.n : n, off = p.embed ? p.win_off : 0;
    const float* surf = ((p.xy_surf && !p.embed) ? p.xy_surf : p.surf) + (size_t)pair * n * n;
    const int pr = pk_i / n, pc = pk_i % n;
    const int w = p.window;
    const int r0 = max(off, pr - w), r1 = min(off + nv - 1, pr + w);
    const int c0 = max(off, pc - w), c1 = min(off + nv - 1, pc + w);
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
    block_sum3(ws, rsum, csum, sh3);
    if (threadIdx.x == 0) {
        const RotState rs = p.rot[pair];
        const double ty_ = rsum / ws, tx_ = csum / ws;
        const double sn = pre_sn, cs = pre_cs;  // published by block_sum3's barriers
        const double tx = cs * tx_ - sn * ty_;
        const double ty = sn * tx_ + cs * ty_;
        if (p.txy_only) {
            p.txy_only[2 * pair] = tx;
            p.txy_only[2 * pair + 1] = ty;
        }
        if (p.out) {
            fscan_pair_result o;
            o.theta = pre_th;
            o.tx = tx;
            o.ty = ty;
            o.theta_hard = rs.hard;
            o.theta_peak = rs.peak;
            o.xy_hard_x = (pc - half) * p.delta;
            o.xy_hard_y = (pr - half) * p.delta;
            o.xy_peak = (double)pk_v;
            o.theta_bin = rs.bin;
            o.xy_row = pr - off;
            o.xy_col = pc - off;
            const int fl = p.chain ? (p.flags[pair] | p.flags[pair + 1]) : p.flags[pair];
            o.status = (fl & 2) ? FSCAN_ERR_MASK_RANGE : ((fl & 1) ? FSCAN_ERR_NONFINITE : FSCAN_OK);
            p.out[pair] = o;
        }
    }
    if (p.embed && p.xy_surf) {  // the reference's nv x nv lag window of the embedded surface
        float* dst = p.xy_surf + (size_t)pair * nv * nv;
        for (int q = threadIdx.x; q < nv * nv; q += kFinThreads)
            dst[q] = surf[(size_t)(off + q / nv) * n + off + q % nv];
    }
}

// band magnitude stage output: tiled [2][N/16][N][8] (f only) -> [N][N/2]
__global__ void k_mag_unpack(Params p) {
    const int n = p.n, w = p.nw;  // half plane u < W = n - n/2
    const int pair = blockIdx.y;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)n * w) return;
    const int vc = (int)(idx / w), u = (int)(idx % w);
    const float2* m = reinterpret_cast<const float2*>(p.mag) + (size_t)pair * p.mag_plane;
    p.mag_out[(size_t)pair * n * w + idx] = tile_at(m, n, vc, u)->x;
}

// K0 in two steps: the cell geometry (fp64 atan2 / sqrt, identical for every
// sweep of a call) once into a table, then a pure gather per sweep.
__global__ void k_polar_taps(int n_az, double res, int n, double delta, fscan_k0::PolarTap* tab) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    tab[idx] = fscan_k0::polar_tap(n_az, res, n, delta, idx / n, idx % n);
}

// PP pairs per thread: the cell's 32-byte tap is read once for all of them (at
// one pair per thread the table's L2 reads, 8 MB per pair at N = 512, were K0's
// largest traffic) and their 8 PP gathers are in flight together. Measured at C3:
// PP = 1 / 2 / 4 / 8 -> 110.9k / 115.1k / 113.3k / 111.5k pairs/s.
#ifndef FSCAN_K0_PP
#define FSCAN_K0_PP 2
#endif
template <int PP>
__global__ void k_polar_to_cart(const float* polar0, const float* polar1, int batch, int n_az, int n_range, int n,
                                const fscan_k0::PolarTap* __restrict__ tab, float* out0, float* out1) {
    const int pair0 = blockIdx.y * PP;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    // both sweeps of every pair from one read of the cell's tap (geometry shared)
    const fscan_k0::PolarTap tp = tab[idx];
    float v0[PP], v1[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) {
        const int pair = pair0 + j < batch ? pair0 + j : batch - 1;  // tail: recompute the last pair (not stored)
        const size_t po = (size_t)pair * n_az * n_range;
        v0[j] = (float)fscan_k0::polar_sample(polar0 + po, n_range, tp);
        v1[j] = polar1 ? (float)fscan_k0::polar_sample(polar1 + po, n_range, tp) : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < PP; ++j) {
        if (pair0 + j < batch) {
            const size_t oo = (size_t)(pair0 + j) * n * n + idx;
            out0[oo] = v0[j];
            if (polar1) out1[oo] = v1[j];
        }
    }
}

// Brute-force correlative search (oracle.cpp:21-67): per (pair, candidate)
// item the hard argmax of its translation surface from K5's block partials
// (strict >, lowest linear index on ties, like score_theta's row-major scan).
__global__ void k_bf_items(Params p, int nparts) {
    const int item = blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= p.batch) return;
    const Partial* pp = p.part + (size_t)item * nparts;
    Partial b = pp[0];
    for (int k = 1; k < nparts; ++k)
        if (pp[k].val > b.val || (pp[k].val == b.val && pp[k].idx < b.idx)) b = pp[k];
    p.bf_items[p.item_base + item] = b;
}

// Winner over the candidates of each pair (strict >: the earlier theta wins
// ties, oracle.cpp:56-58) and its pose: t = R(theta) (col - half, row - half) delta.
// np: pitch of the surface the partial indices refer to, off: offset of the
// reference's n x n lag window in it (0 unless the grid is embedded, §3.9)
__global__ void k_bf_final(const Partial* items, const double* thetas, int nth, int batch, int n, int np,
                           int off, double delta, fscan_bf_result* out) {
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= batch) return;
    const Partial* it = items + (size_t)pair * nth;
    int w = 0;
    for (int k = 1; k < nth; ++k)
        if (it[k].val > it[w].val) w = k;
    const int half = (n - 1) / 2;
    const int idx = it[w].idx == 0x7fffffff ? off * np + off : it[w].idx;  // all-NaN: first cell
    const int row = idx / np - off, col = idx % np - off;
    const double theta = thetas[w];
    const double dx = (col - half) * delta, dy = (row - half) * delta;
    double sn, cs;
    sincos(theta, &sn, &cs);  // rotate_vec (geometry.cpp:31-35)
    const double two_pi = 6.283185307179586, pi = 3.141592653589793;
    double th = fmod(theta, two_pi);  // normalize_angle (geometry.cpp:9-14)
    if (th <= -pi) th += two_pi;
    if (th > pi) th -= two_pi;
    fscan_bf_result o;
    o.theta = th;
    o.tx = cs * dx - sn * dy;
    o.ty = sn * dx + cs * dy;
    o.score = (double)it[w].val;
    o.theta_index = w;
    o.xy_row = row;
    o.xy_col = col;
    o.status = isfinite(it[w].val) ? FSCAN_OK : FSCAN_ERR_NONFINITE;
    out[pair] = o;
}

// A/B knob: FSCAN_CARVEOUT=<percent> asks for that shared-memory carveout
// (cudaFuncAttributePreferredSharedMemoryCarveout) for the pipeline stages whose
// bit is set in FSCAN_CARVEOUT_MASK (bit = Stage, default all); unset = the
// driver's choice per kernel.
enum Stage { kStRotRows, kStRotCols, kStRotGather, kStRotPolar, kStXRows, kStXCols, kStXOut, kStFin };
inline int carveout_for(int stage) {
    static const int pct = [] { const char* e = getenv("FSCAN_CARVEOUT"); return e ? atoi(e) : -1; }();
    static const int mask = [] { const char* e = getenv("FSCAN_CARVEOUT_MASK"); return e ? (int)strtol(e, nullptr, 0) : 0xff; }();
    return (pct >= 0 && ((mask >> stage) & 1)) ? pct : -1;
}
template <typename K>
cudaError_t set_carveout(K kernel, int stage) {
    const int pct = carveout_for(stage);
    return pct < 0 ? cudaSuccess : cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes, int stage = -1) {
    if (stage >= 0) {
        cudaError_t e = set_carveout(kernel, stage);
        if (e != cudaSuccess) return e;
    }
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

// Launch of a pipeline kernel (one that starts with pdl_enter / pdl_wait):
// with programmatic stream serialisation when the context asks for it.
template <typename... KA, typename... A>
cudaError_t launch_k(void (*kernel)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, const Params& p,
                     A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = p.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int N>
cudaError_t rot_rows(const Params& p, cudaStream_t s) {
    const size_t sm = (size_t)RowG<N>::FLOATS * sizeof(float);
    cudaError_t e = set_smem(k_rot_rows<N>, sm, kStRotRows);
    if (e != cudaSuccess) return e;
    return launch_k(k_rot_rows<N>, dim3(N / RowG<N>::PER_CTA, p.batch), dim3(kRowThreads), sm, s, p, p);
}

template <int N>
cudaError_t rot_cols(const Params& p, cudaStream_t s) {
    constexpr int U = k1b_u<N>();
    const size_t sm = k1b_smem_floats<N>() * sizeof(float);
    cudaError_t e = set_smem(k_rot_cols<N>, sm, kStRotCols);
    if (e != cudaSuccess) return e;
    return launch_k(k_rot_cols<N>, dim3(p.zcols / U, p.batch), dim3(N / 16 * 2 * U), sm, s, p, p);
}

template <int N>
cudaError_t xlat_rows(const Params& p, cudaStream_t s) {
    using X = XRowGeom<N>;
    const dim3 grid(N / X::ROWS, p.batch);
    auto go = [&](auto kernel) {
        cudaError_t e = set_smem(kernel, X::SMEM, kStXRows);
        if (e != cudaSuccess) return e;
        return launch_k(kernel, grid, dim3(kXThreads), X::SMEM, s, p, p);
    };
    if (p.src_div != 1)  // exhaustive search
        return p.embed ? go(k_xlat_rows<N, true, true>) : go(k_xlat_rows<N, true, false>);
    if (p.embed) return go(k_xlat_rows<N, false, true>);
    if (p.gtex && p.gt == p.gtex_base) return go(k_xlat_rows<N, false, false, true>);  // the lane's own g~
    return go(k_xlat_rows<N, false, false>);
}

template <int N>
cudaError_t xlat_cols(const Params& p, cudaStream_t s) {
    using X = XColGeom<N>;
    constexpr int H = 3 * N / 4;
    const dim3 grid(X::MERGE ? (X::NBLOCKS + X::NBLK - 1) / X::NBLK : (H + 1 + X::COLS - 1) / X::COLS, p.batch);
    constexpr size_t SMEM = X::MERGE ? X::SMEM_MERGE : X::SMEM;
    auto go = [&](auto kernel) {
        cudaError_t e = set_smem(kernel, SMEM, kStXCols);
        if (e != cudaSuccess) return e;
        return launch_k(kernel, grid, dim3(X::THREADS), SMEM, s, p, p);
    };
    if constexpr (X::MIN_BLOCKS > 0)
        return go(k_xlat_cols_mb<N, (X::MIN_BLOCKS > 0 ? X::MIN_BLOCKS : 1)>);
    else
        return go(k_xlat_cols<N>);
}

template <int N>
cudaError_t xlat_win(const Params& p, cudaStream_t s);

template <int N>
cudaError_t xlat_out(const Params& p, cudaStream_t s) {
    using X = XOutGeom<N>;
    const dim3 grid(N / X::ROWS, p.batch);
    auto go = [&](auto kernel) {
        cudaError_t e = set_smem(kernel, X::SMEM, kStXOut);
        if (e != cudaSuccess) return e;
        return launch_k(kernel, grid, dim3(X::THREADS), X::SMEM, s, p, p);
    };
    if (p.embed) return go(k_xlat_out<N, true>);
    return xlat_win_pass(p) ? go(k_xlat_out<N, false, kOutMax>) : go(k_xlat_out<N, false>);
}

template <int N>
cudaError_t xlat_win(const Params& p, cudaStream_t s) {
    using X = XOutGeom<N>;
    constexpr int NB = N / X::ROWS;
    // row blocks a window of 2w + 1 rows can touch
    const int nb = std::min(NB, (2 * p.window + X::ROWS - 1) / X::ROWS + 1);
    cudaError_t e = set_smem(k_xlat_out<N, false, kOutWin>, X::SMEM, kStXOut);
    if (e != cudaSuccess) return e;
    return launch_k(k_xlat_out<N, false, kOutWin>, dim3(nb, p.batch), dim3(X::THREADS), X::SMEM, s, p, p);
}

}  // namespace

// Two-pass K5 (kOutMax + kOutWin) whenever no caller reads the full surface:
// not for embedded grids (K6 copies their lag window out of it), requested
// xy surfaces or the exhaustive search (block maxima only)
bool xlat_win_pass(const Params& p) {
    return FSCAN_K5_TWO_PASS && p.np >= FSCAN_K5_TWO_PASS_MIN_N && !p.embed && !p.xy_surf && !p.skip_surface;
}

int rows_per_block_out(int n) {
    switch (n) {
        case 64: return XOutGeom<64>::ROWS;
        case 128: return XOutGeom<128>::ROWS;
        case 256: return XOutGeom<256>::ROWS;
        case 512: return XOutGeom<512>::ROWS;
        case 1024: return XOutGeom<1024>::ROWS;
        default: return 1;
    }
}

cudaError_t launch_rot_rows(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, rot_rows) }
cudaError_t launch_rot_cols(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.n, rot_cols) }
cudaError_t launch_xlat_rows(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.np, xlat_rows) }
cudaError_t launch_xlat_cols(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.np, xlat_cols) }
cudaError_t launch_xlat_out(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.np, xlat_out) }
cudaError_t launch_xlat_win(const Params& p, cudaStream_t s) { FSCAN_DISPATCH_N(p.np, xlat_win) }

cudaError_t launch_rot_gather(const Params& p, cudaStream_t s) {
    if (p.n_theta == 1) return cudaSuccess;
    if (FSCAN_K2A_PB > 1 && !p.chain) {
        constexpr int PB = FSCAN_K2A_PB > 1 ? FSCAN_K2A_PB : 2;
        auto go = [&](auto kernel, int rp) {
            if (cudaError_t e = set_carveout(kernel, kStRotGather); e != cudaSuccess) return e;
            const int az = kGatherThreads / rp;  // azimuths per CTA
            return launch_k(kernel, dim3((p.n_theta + az - 1) / az, (p.batch + PB - 1) / PB), dim3(kGatherThreads),
                            0, s, p, p);
        };
        if (p.n <= 256) return go(k_rot_gather_multi<PB, FSCAN_K2A_RP_SMALL>, FSCAN_K2A_RP_SMALL);
        return go(k_rot_gather_multi<PB, 4>, 4);
    }
    return launch_k(k_rot_gather, dim3((p.n_theta + kGatherThreads / 4 - 1) / (kGatherThreads / 4), p.batch),
                    dim3(kGatherThreads), 0, s, p, p);
}

// CTAs per pair for K2b: one when the batch fills the GPU, else up to 16
#ifndef FSCAN_K2B_FUSE_FIN
#define FSCAN_K2B_FUSE_FIN 1  // split K2b: the pair's last CTA runs the argmaxes (no k_rot_polar_fin launch)
#endif
#ifndef FSCAN_K2B_BIG_SPLIT
#define FSCAN_K2B_BIG_SPLIT 1  // CTAs per pair for batches that fill the GPU
#endif
int polar_split(int batch, int nt) {
    if (nt <= 1) return 1;
    if (batch >= FSCAN_K2B_SPLIT_BELOW) return FSCAN_K2B_BIG_SPLIT;
    return std::min(16, (148 + batch - 1) / batch);
}

cudaError_t launch_rot_polar(const Params& p, cudaStream_t s) {
    const int S = polar_split(p.batch, p.n_theta);
    if (S > 1) {
        const int blocks = (p.n_theta + kLags - 1) / kLags, per = (blocks + S - 1) / S;
        const size_t fm0 = (size_t)(2 * p.n_theta + 32) * sizeof(double) + 32 * sizeof(int);  // polar_finish
        const int fuse = FSCAN_K2B_FUSE_FIN && p.polar_cnt != nullptr;
        const size_t sm = std::max((size_t)(p.L + bx_len(p.L, p.n_theta) +
                                            (size_t)polar_parts(p.n_theta) * per * kLags) * sizeof(double),
                                   fuse ? fm0 : (size_t)0);
        cudaError_t e = set_smem(k_rot_polar_part, sm, kStRotPolar);
        if (e != cudaSuccess) return e;
        if ((e = launch_k(k_rot_polar_part, dim3(p.batch * S), dim3(kPolarThreads), sm, s, p, p, S, fuse)) !=
                cudaSuccess ||
            fuse)
            return e;
        const size_t fm = (size_t)(2 * p.n_theta + 32) * sizeof(double) + 32 * sizeof(int);
        if ((e = set_smem(k_rot_polar_fin, fm)) != cudaSuccess) return e;
        return launch_k(k_rot_polar_fin, dim3(p.batch), dim3(kPolarThreads), fm, s, p, p);
    }
    const size_t sm = (size_t)(p.L + bx_len(p.L, p.n_theta) + p.n_theta * (1 + polar_parts(p.n_theta)) + 32) *
                          sizeof(double) +
                      32 * sizeof(int);
    cudaError_t e = set_smem(k_rot_polar, sm, kStRotPolar);
    if (e != cudaSuccess) return e;
    return launch_k(k_rot_polar, dim3(p.batch), dim3(kPolarThreads), sm, s, p, p);
}

cudaError_t launch_theta_in(const Params& p, cudaStream_t s) {
    k_theta_in<<<(p.batch + 127) / 128, 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Params& p, cudaStream_t s) {
    return launch_k(k_finalize, dim3(p.batch), dim3(kFinThreads), 0, s, p, p, p.np / rows_per_block_out(p.np));
}

cudaError_t launch_mag_unpack(const Params& p, cudaStream_t s) {
    const size_t total = (size_t)p.n * p.nw;
    k_mag_unpack<<<dim3((unsigned)((total + 255) / 256), p.batch), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_bf_items(const Params& p, cudaStream_t s) {
    k_bf_items<<<(p.batch + 127) / 128, 128, 0, s>>>(p, p.np / rows_per_block_out(p.np));
    return cudaGetLastError();
}

// Copies count n x n grids into the top-left of zeroed np x np grids.
__global__ void k_embed(const float* __restrict__ src, int n, int np, float* __restrict__ dst) {
    const int b = blockIdx.y;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
        dst[(size_t)b * np * np + (size_t)(e / n) * np + e % n] = src[(size_t)b * n * n + e];
}

cudaError_t launch_embed(const float* src, int count, int n, int np, float* dst, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    k_embed<<<dim3(64, count), 256, 0, s>>>(src, n, np, dst);
    return cudaGetLastError();
}

cudaError_t launch_bf_final(const Partial* items, const double* thetas, int n_thetas, int batch, int n,
                                  int np, int off, double delta, fscan_bf_result* out, cudaStream_t s) {
    k_bf_final<<<(batch + 127) / 128, 128, 0, s>>>(items, thetas, n_thetas, batch, n, np, off, delta, out);
    return cudaGetLastError();
}

size_t polar_tap_bytes(int n) { return sizeof(fscan_k0::PolarTap) * (size_t)n * n; }

cudaError_t launch_polar_taps(int n_az, double range_res, int n, double delta, void* tab, cudaStream_t stream) {
    const int total = n * n;
    k_polar_taps<<<(total + 255) / 256, 256, 0, stream>>>(n_az, range_res, n, delta,
                                                           static_cast<fscan_k0::PolarTap*>(tab));
    return cudaGetLastError();
}

cudaError_t launch_polar_to_cart(const float* d_polar0, const float* d_polar1, int batch, int n_az,
                                 int n_range, double range_res, int n, double delta, float* d_out0,
                                 float* d_out1, cudaStream_t stream, const void* tab) {
    const int total = n * n;
    void* own = nullptr;
    if (!tab) {  // no cached table: build one for this call
        cudaError_t e = cudaMallocAsync(&own, polar_tap_bytes(n), stream);
        if (e != cudaSuccess) return e;
        e = launch_polar_taps(n_az, range_res, n, delta, own, stream);
        if (e != cudaSuccess) return e;
        tab = own;
    }
    constexpr int PP = FSCAN_K0_PP;
    k_polar_to_cart<PP><<<dim3((unsigned)((total + 255) / 256), (batch + PP - 1) / PP), 256, 0, stream>>>(
        d_polar0, d_polar1, batch, n_az, n_range, n, static_cast<const fscan_k0::PolarTap*>(tab), d_out0, d_out1);
    cudaError_t e = cudaGetLastError();
    if (own) cudaFreeAsync(own, stream);
    return e;
}

}  // namespace fscan_detail
