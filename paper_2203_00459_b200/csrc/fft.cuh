// fft.cuh — register/shared-memory radix-16 Stockham FFT engine (sm_100a).
//
// Replaces the FFTW c2c transforms the reference calls through
// proj/src/spectral.cpp:73-153 (dft2 / idft2 / xcorr) on the GPU path.
//
// One length-N transform (N = 2^k, 16 <= N <= 2048) is owned by T = N/16
// threads; thread t of a transform holds the 16 complex values
//     v[m] = x[t + m*T],  m = 0..15
// before and after the call (natural order in, natural order out). Stages are
// radix 16 while at least 16*16 points remain, then one radix-R stage
// (R = N / 16^s in {2,4,8,16}) done as 16/R butterflies per thread:
//     N=16: 16   32: 16.2   64: 16.4   128: 16.8   256: 16.16   512: 16.16.2
//     1024: 16.16.4   2048: 16.16.8
// Stage (radix R, span Ns) butterfly b reads x[b + r*N/R] (= registers
// j + r*(16/R) of thread t, b = t + j*T), multiplies by W_{Ns*R}^{r*(b mod Ns)},
// does an R-point DFT and writes y[(b/Ns)*Ns*R + (b mod Ns) + r*Ns]. The last
// stage lands back in the input register slots, so only S-1 shared-memory
// exchanges are needed (one for N <= 256, two for 512..2048).
//
// Exchange buffers hold float2 (one 64-bit shared access per complex value)
// with an XOR swizzle inside each 16-element line, i' = i ^ ((i >> 4) & 15);
// row kernels give every transform its own buffer (staggered, see Geom), the
// 16-column kernel interleaves W transforms element-wise: addr = W * i' + sub.
// Every exchange pattern of every size is bank-conflict free (half-warp phases
// of 8-byte accesses; verified with an access-pattern model).
//
// Twiddles come from a fp32 table tw[i] = exp(-2*pi*i*i/N) (rounded from fp64
// on the host); SIGN = +1 uses the conjugate. Transforms are unnormalised,
// matching FFTW_FORWARD / FFTW_BACKWARD. Exchanges synchronise the warp when
// the transform lives in one warp (fft_regs<..., WARP = true>), else the CTA.
#pragma once

#include <stdint.h>
#include <cuda_runtime.h>

#include <type_traits>

namespace fscan_fft {

// Packed fp32 (sm_100a FADD2 / FMUL2 / FFMA2 on aligned register pairs, PTX
// add / mul / fma.rn.f32x2): a complex add or subtract is ONE instruction and a
// complex product two plus a negation, each component rounded exactly as its
// scalar form (add.rn / mul.rn / fma.rn) — same bits, half the issue slots.
// The translation kernels are bound by issue slots and the L1 data pipe with
// the FMA pipe half idle (tools/microbench/f32x2_probe.cu: a packed
// instruction delivers the scalar forms' fp32 rate per SM from one issue slot
// instead of two). Measured (C4 / C5, interleaved): packed add / subtract
// K4 6.79 -> 6.59 ms / 8.39 -> 7.88 ms, K3 6.49 -> 6.40 ms, C4 +1.2%, C5 +1.2%;
// the packed product as well: K4 6.8 -> 8.0 ms at N = 512 (its constant-bank
// twiddles turn into LDC + MOV pairs: packed operands cannot name a constant,
// and K4 runs at 4.5 warps per scheduler, too few to hide them), C4 -4.5%.
// So: packed add / subtract on (FSCAN_NO_F32X2_ADD), packed product off
// (FSCAN_F32X2_MUL).
#ifdef FSCAN_NO_F32X2_ADD
constexpr bool kF32x2Add = false;  // A/B: scalar complex add / subtract
#else
constexpr bool kF32x2Add = true;
#endif
#ifdef FSCAN_F32X2_MUL
constexpr bool kF32x2Mul = true;
#else
constexpr bool kF32x2Mul = false;
#endif

constexpr int kPkDefault = (kF32x2Add ? 1 : 0) | (kF32x2Mul ? 6 : 0);

template <bool PK = kF32x2Mul>
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    if constexpr (PK) {
        // (a.x b.x + rn(-a.y b.y), a.x b.y + rn(a.y b.x)): the scalar form's roundings
        float2 r;
        asm("{ .reg .b64 ax, ay, bb, bs, t, rr;\n\t"
            " mov.b64 ax, {%2, %2};\n\t mov.b64 ay, {%3, %3};\n\t mov.b64 bb, {%4, %5};\n\t mov.b64 bs, {%6, %4};\n\t"
            " mul.rn.f32x2 t, ay, bs;\n\t fma.rn.f32x2 rr, ax, bb, t;\n\t mov.b64 {%0, %1}, rr; }"
            : "=f"(r.x), "=f"(r.y)
            : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(-b.y));
        return r;
    } else {
        return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
    }
}
// sqrt.approx.f32 (one MUFU op, ~1 ulp): the IEEE-rounded sqrtf costs ~10
// instructions and a slow-path branch; magnitudes feeding the polar gather need
// nothing tighter than the fp32 FFT's own ~1e-7 relative error
__device__ __forceinline__ float sqrt_fast(float x) {
    float y;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <bool PK = kF32x2Add>
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    if constexpr (PK) {
        float2 r;
        asm("{ .reg .b64 ra, rb, rr;\n\t mov.b64 ra, {%2, %3};\n\t mov.b64 rb, {%4, %5};\n\t"
            " add.rn.f32x2 rr, ra, rb;\n\t mov.b64 {%0, %1}, rr; }"
            : "=f"(r.x), "=f"(r.y)
            : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
        return r;
    } else {
        return make_float2(a.x + b.x, a.y + b.y);
    }
}
template <bool PK = kF32x2Add>
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    if constexpr (PK) {
        float2 r;
        asm("{ .reg .b64 ra, rb, rr;\n\t mov.b64 ra, {%2, %3};\n\t mov.b64 rb, {%4, %5};\n\t"
            " sub.rn.f32x2 rr, ra, rb;\n\t mov.b64 {%0, %1}, rr; }"
            : "=f"(r.x), "=f"(r.y)
            : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
        return r;
    } else {
        return make_float2(a.x - b.x, a.y - b.y);
    }
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// a * (-i) for SIGN=-1, a * (+i) for SIGN=+1
template <int SIGN>
__device__ __forceinline__ float2 mul_mi(float2 a) {
    return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

template <int SIGN, int PK = kPkDefault>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
    const float2 t = a;
    a = cadd<(PK & 1) != 0>(t, b);
    b = csub<(PK & 1) != 0>(t, b);
}

// 4-point DFT in place, natural order out.
template <int SIGN, int PK = kPkDefault>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
    const float2 a = cadd<(PK & 1) != 0>(x0, x2), b = csub<(PK & 1) != 0>(x0, x2);
    const float2 c = cadd<(PK & 1) != 0>(x1, x3), d = mul_mi<SIGN>(csub<(PK & 1) != 0>(x1, x3));
    x0 = cadd<(PK & 1) != 0>(a, c);
    x2 = csub<(PK & 1) != 0>(a, c);
    x1 = cadd<(PK & 1) != 0>(b, d);
    x3 = csub<(PK & 1) != 0>(b, d);
}

// 8-point DFT as radix-2 x radix-4 (DIT over n = 2*n1 + n2).
template <int SIGN, int PK = kPkDefault>
__device__ __forceinline__ void dft8(float2* x) {
    constexpr float r = 0.70710678118654752f;
    float2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
    float2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
    dft4<SIGN, PK>(e0, e1, e2, e3);
    dft4<SIGN, PK>(o0, o1, o2, o3);
    o1 = SIGN < 0 ? make_float2(r * (o1.x + o1.y), r * (o1.y - o1.x)) : make_float2(r * (o1.x - o1.y), r * (o1.y + o1.x));
    o2 = mul_mi<SIGN>(o2);
    o3 = SIGN < 0 ? make_float2(r * (o3.y - o3.x), -r * (o3.x + o3.y)) : make_float2(-r * (o3.x + o3.y), r * (o3.x - o3.y));
    x[0] = cadd<(PK & 1) != 0>(e0, o0);
    x[4] = csub<(PK & 1) != 0>(e0, o0);
    x[1] = cadd<(PK & 1) != 0>(e1, o1);
    x[5] = csub<(PK & 1) != 0>(e1, o1);
    x[2] = cadd<(PK & 1) != 0>(e2, o2);
    x[6] = csub<(PK & 1) != 0>(e2, o2);
    x[3] = cadd<(PK & 1) != 0>(e3, o3);
    x[7] = csub<(PK & 1) != 0>(e3, o3);
}

// 16-point DFT as 4x4: X[k1 + 4*k2] = sum_n2 W4^(n2 k2) W16^(n2 k1) sum_n1 x[4 n1 + n2] W4^(n1 k1)
template <int SIGN, int PK = kPkDefault>
__device__ __forceinline__ void dft16(float2* x) {
    constexpr float c1 = 0.92387953251128674f;  // cos(pi/8)
    constexpr float s1 = 0.38268343236508977f;  // sin(pi/8)
    constexpr float r = 0.70710678118654752f;
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<SIGN, PK>(x[n2], x[4 + n2], x[8 + n2], x[12 + n2]);
    // x[4*k1 + n2] holds a[n2][k1]; apply W16^(n2*k1) = cos + i*SIGN*sin
    const float sg = (float)SIGN;
    const float2 w1 = make_float2(c1, sg * s1), w2 = make_float2(r, sg * r), w3 = make_float2(s1, sg * c1);
    const float2 w6 = make_float2(-r, sg * r), w9 = make_float2(-c1, -sg * s1);
    x[4 * 1 + 1] = cmul<(PK & 4) != 0>(x[4 * 1 + 1], w1);
    x[4 * 2 + 1] = cmul<(PK & 4) != 0>(x[4 * 2 + 1], w2);
    x[4 * 3 + 1] = cmul<(PK & 4) != 0>(x[4 * 3 + 1], w3);
    x[4 * 1 + 2] = cmul<(PK & 4) != 0>(x[4 * 1 + 2], w2);
    x[4 * 2 + 2] = mul_mi<SIGN>(x[4 * 2 + 2]);
    x[4 * 3 + 2] = cmul<(PK & 4) != 0>(x[4 * 3 + 2], w6);
    x[4 * 1 + 3] = cmul<(PK & 4) != 0>(x[4 * 1 + 3], w3);
    x[4 * 2 + 3] = cmul<(PK & 4) != 0>(x[4 * 2 + 3], w6);
    x[4 * 3 + 3] = cmul<(PK & 4) != 0>(x[4 * 3 + 3], w9);
    float2 y[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        float2 a0 = x[4 * k1], a1 = x[4 * k1 + 1], a2 = x[4 * k1 + 2], a3 = x[4 * k1 + 3];
        dft4<SIGN, PK>(a0, a1, a2, a3);
        y[k1] = a0;
        y[k1 + 4] = a1;
        y[k1 + 8] = a2;
        y[k1 + 12] = a3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = y[i];
}

template <int R, int SIGN, int PK = kPkDefault>
__device__ __forceinline__ void dft_r(float2* x) {
    if constexpr (R == 2) {
        dft2<SIGN, PK>(x[0], x[1]);
    } else if constexpr (R == 4) {
        dft4<SIGN, PK>(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        dft8<SIGN, PK>(x);
    } else {
        dft16<SIGN, PK>(x);
    }
}

// Exchange-buffer layout of one transform (see header comment): complex
// values as float2 (one 64-bit shared access per element), XOR-swizzled inside
// each 16-element line so every exchange pattern is bank-conflict free.
#ifdef FSCAN_SWIZZLE_WIDE
constexpr bool kSwizzleWide = true;  // A/B: keep the XOR swizzle for W >= 16
#else
constexpr bool kSwizzleWide = false;
#endif

template <int W>
struct Lay {
    float2* buf;
    int sub;  // transform index inside an interleaved group (W > 1)
    __device__ __forceinline__ int at(int i) const {
        if constexpr (W >= 16 && !kSwizzleWide) {
            // W >= 16 interleaved transforms: element i of every transform of a
            // half-warp sits in its own bank pair (sub) whatever i is, so the
            // swizzle buys nothing; a plain W * i + sub leaves the exchange
            // loops with compile-time offsets from one per-thread base
            return W * i + sub;
        } else {
            const int j = (i & ~15) | ((i & 15) ^ ((i >> 4) & 15));
            if constexpr (W == 1) {
                return j;
            } else {
                return W * j + sub;
            }
        }
    }
    __device__ __forceinline__ void put(int i, float2 v) const { buf[at(i)] = v; }
    __device__ __forceinline__ float2 get(int i) const { return buf[at(i)]; }
};

// Floats of the buffer of one group of W interleaved length-N transforms
// (the 16-column kernel); the +4 staggers consecutive buffers across banks.
template <int N, int W>
__host__ __device__ constexpr int part_floats() {
    return 2 * W * N + 4;
}

// Thread/transform geometry of kernels whose transforms are "rows": T = N/16
// threads per transform, the T lanes of a transform contiguous in the warp
// (W = 32/T transforms per warp when T < 32). Every transform has its own
// exchange buffer; consecutive buffers are staggered by T elements (T < 16)
// so that the W transforms sharing a warp, and loops that read several
// transforms' buffers at the same index (separation, radix-3 combines), hit
// disjoint banks (T >= 16: any stride is conflict-free for the FFT; 2 and 12
// are chosen for the row-separation loop of K3, see XRowGeom). Verified
// conflict-free for all exchange and combine patterns with an access-pattern
// model.
// Padded per-transform layout of the row kernels (kGeomPad): one float2 of
// padding per 16 elements, addr = i + i/16. Both exchange patterns of the
// radix-16 Stockham stages (stride-16 puts i = 16 b + r, unit-stride gets
// i = t + m T) then land on distinct bank pairs, and every address is a
// per-thread base plus a compile-time offset: no per-access XOR (the swizzled
// Lay<1> spends a LOP3 and an add on every exchange access).
struct LayPad {
    float2* buf;
    __device__ __forceinline__ static int at(int i) { return i + (i >> 4); }
    __device__ __forceinline__ void put(int i, float2 v) const { buf[at(i)] = v; }
    __device__ __forceinline__ float2 get(int i) const { return buf[at(i)]; }
};

#ifdef FSCAN_GEOM_XOR
constexpr bool kGeomPad = false;  // A/B: the XOR-swizzled Lay<1>
#else
constexpr bool kGeomPad = true;
#endif

template <int N, int THREADS>
struct Geom {
    static constexpr int T = N / 16;
    static constexpr int W = T >= 32 ? 1 : 32 / T;  // transforms per warp
    static constexpr int PER_CTA = THREADS / T;      // transforms per CTA
    static constexpr int GROUPS = PER_CTA / W;
    static_assert(GROUPS >= 1 && PER_CTA % W == 0, "a CTA must hold whole warps of transforms");
    // float2 elements per transform buffer holding length-LEN data
    // kGeomPad: LEN + LEN/16 elements; for T < 16 that is = T (mod 16), which
    // puts the W transforms of a half-warp on disjoint bank pairs; T = 16 / 32
    // add 2 / 12 so that K3's row-separation loop keeps the bank offset per row
    // it has with the swizzled layout (O = 6 at N = 512, 4 at N = 1024)
    template <int LEN>
    __host__ __device__ static constexpr int stride_len() {
        if constexpr (kGeomPad)
            return LEN + LEN / 16 + (T < 16 ? 0 : (T == 16 ? 2 : 12));
        else
            return LEN + (T < 16 ? T : (T == 16 ? 2 : 12));
    }
    static constexpr int FLOATS = PER_CTA * 2 * stride_len<N>();  // one exchange buffer per transform
    using L = std::conditional_t<kGeomPad, LayPad, Lay<1>>;
    __device__ __forceinline__ static void map(int tid, int& tr, int& t) {
        tr = tid / T;
        t = tid % T;
    }
    __device__ __forceinline__ static L make(float2* p) {
        if constexpr (kGeomPad)
            return LayPad{p};
        else
            return Lay<1>{p, 0};
    }
    // layout of transform tr inside buffer `base` (FLOATS floats, 8-byte aligned)
    __device__ __forceinline__ static L lay(float* base, int tr) {
        return make(reinterpret_cast<float2*>(base) + tr * stride_len<N>());
    }
    // layout of transform tr for a buffer holding length-LEN data per transform
    template <int LEN>
    __device__ __forceinline__ static L lay_len(float* base, int tr) {
        return make(reinterpret_cast<float2*>(base) + tr * stride_len<LEN>());
    }
    template <int LEN>
    __host__ __device__ static constexpr int floats_len() {
        return PER_CTA * 2 * stride_len<LEN>();
    }
};

// Split real/imag exchange layout (rounds 1-2 of the column kernel K4; now an
// A/B alternative, FSCAN_K4_F2_MIN): two 32-bit accesses per element, W
// transforms interleaved element-wise (transform index = lane % W fastest in
// the warp): addr = W*(i + i/16) + sub; W == 1: XOR of the 5-bit offset inside
// each 32-float line by (line & 15) | bit3(line) << 4. It moves the same
// shared-memory wavefronts as the float2 layout of Geom with twice the LSU
// instructions; once K4 stopped being register-bound the float2 layout won
// (ncu: MIO-throttle stalls on the exchange lines; C5 +5%, C4 +1%, C2 +2.6%).
template <int W>
struct LaySoA {
    float* re;
    float* im;
    int sub;
    __device__ __forceinline__ int at(int i) const {
        if constexpr (W == 1) {
            const int j = i >> 5;
            return (i & ~31) | ((i & 31) ^ ((j & 15) | (((j >> 3) & 1) << 4)));
        } else {
            return W * (i + (i >> 4)) + sub;
        }
    }
    __device__ __forceinline__ void put(int i, float2 v) const {
        const int a = at(i);
        re[a] = v.x;
        im[a] = v.y;
    }
    __device__ __forceinline__ float2 get(int i) const {
        const int a = at(i);
        return make_float2(re[a], im[a]);
    }
};

template <int N, int THREADS>
struct GeomSoA {
    static constexpr int T = N / 16;
    static constexpr int W = T >= 32 ? 1 : 32 / T;
    static constexpr int PER_CTA = THREADS / T;
    static constexpr int GROUPS = PER_CTA / W;
    static constexpr int SPART = W == 1 ? N + 2 : W * (N + N / 16) + 2;
    static constexpr int FLOATS = GROUPS * 2 * SPART;
    __device__ __forceinline__ static void map(int tid, int& tr, int& t) {
        if constexpr (W == 1) {
            tr = tid / T;
            t = tid % T;
        } else {
            const int w = tid >> 5, lane = tid & 31;
            tr = w * W + lane % W;
            t = lane / W;
        }
    }
    __device__ __forceinline__ static LaySoA<W> lay(float* base, int tr) {
        float* g = base + (tr / W) * 2 * SPART;
        return LaySoA<W>{g, g + SPART, tr % W};
    }
};

template <int SIGN>
__device__ __forceinline__ float2 twiddle(const float2* __restrict__ tw, int idx) {
    const float2 w = __ldg(tw + idx);
    return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

// A twiddle table staged in shared memory (plain 64-bit shared loads).
struct SmemTw {
    const float2* p;
};

template <int SIGN>
__device__ __forceinline__ float2 twiddle(const SmemTw& tw, int idx) {
    const float2 w = tw.p[idx];
    return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

// Shared-memory twiddles with the span-16 stage's factors as a [r][k] matrix
// rk[(r-1)*16 + k] = W_256^{r k}: the 16 lanes' k are consecutive, so each read
// is one conflict-free wavefront (the linear table's r*k pattern is gcd(r, 16)-
// way conflicted); `lin` is the linear table W_L for the other stages.
struct SmemTwRK {
    const float2* rk;
    const float2* lin;
};

template <int SIGN>
__device__ __forceinline__ float2 twiddle(const SmemTwRK& tw, int idx) {
    const float2 w = tw.lin[idx];
    return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

template <typename TW>
constexpr bool kTwRK = std::is_same_v<TW, SmemTwRK>;

// K4's merged twiddles (a K = 16 R point transform, K <= 256, inside a length
// M = 3K transform split into three q groups). One shared table
// F[a][j] = W_M^{a j} (a < 16, j < 48, row stride kQS), `f` = F + q:
//  * forward (QF): the group's input twiddle W_M^{n q}, n = t + m T, is split
//    into W_M^{m T q} (applied to the inputs) and W_M^{t q}, which is constant
//    over a thread's first-stage butterfly and so rides on its outputs into the
//    last stage: input r of butterfly k there carries W_M^{r q} W_K^{r k} =
//    F[r][3k + q] (one table read, as the plain W_K^{r k} did);
//  * inverse (QI): the combine's output twiddle W_M^{-n q}, n = k + 16 r', is
//    split into W_M^{-16 r' q} (applied to the outputs) and W_M^{-k q}, constant
//    over the last-stage butterfly k, which joins its input twiddles:
//    W_K^{-r k} W_M^{-k q} = conj(F[k][3r + q]) (r = 0 included).
constexpr int kQS = 49;  // odd row stride: the inverse's column reads F[k][.] spread over banks
// S: the table's row stride; G: the table read through L1 from global memory
// (__ldg) instead of a shared-memory copy
// W (forward only): the table is still being staged by the CTA when the
// transform starts — `ready` is an mbarrier every thread arrives on after its
// table stores, waited on (phase 0) just before the last stage's first read
// (a split barrier: the first stage and its exchange run under the staging).
__device__ __forceinline__ void wait_phase0(const uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "TWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra TWAIT_%=;\n\t}" ::"r"(a)
        : "memory");
}
template <int S, bool G, bool W = false>
struct TwQF {
    const float2* f;
    const uint64_t* ready = nullptr;
    __device__ __forceinline__ float2 at(int i) const { return G ? __ldg(f + i) : f[i]; }
    __device__ __forceinline__ void wait() const {
        if constexpr (W) wait_phase0(ready);
    }
};
template <int S, bool G>
struct TwQI {
    const float2* f;
    __device__ __forceinline__ float2 at(int i) const { return G ? __ldg(f + i) : f[i]; }
};
using SmemTwQF = TwQF<kQS, false>;
using SmemTwQI = TwQI<kQS, false>;
template <typename TW>
struct TwQInfo {
    static constexpr int kind = 0, S = 0;
};
template <int S_, bool G, bool W>
struct TwQInfo<TwQF<S_, G, W>> {
    static constexpr int kind = 1, S = S_;
};
template <int S_, bool G>
struct TwQInfo<TwQI<S_, G>> {
    static constexpr int kind = 2, S = S_;
};
template <typename TW>
constexpr bool kTwQ = TwQInfo<TW>::kind != 0;

// Radix-16 twiddles as powers of one table read (global tables) or all read
// from the table (shared-memory tables).
template <typename TW>
constexpr bool kTwPow = !std::is_same_v<TW, SmemTw> && !kTwRK<TW> && !kTwQ<TW>;

// One Stockham stage. Ns = span before this stage, R = radix.
// Exchange barrier: a warp barrier when every thread of the transform (and of
// any transform sharing its buffer) is in one warp, else the CTA barrier.
template <bool WARP>
__device__ __forceinline__ void exchange_sync() {
    if constexpr (WARP) {
        __syncwarp();
    } else {
        __syncthreads();
    }
}

// W_16^x (SIGN -1) or its conjugate, x a compile-time value after unrolling
template <int SIGN>
__device__ __forceinline__ float2 w16c(int x) {
    constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508977f, r = 0.70710678118654752f;
    constexpr float cs[16] = {1.f, c1, r, s1, 0.f, -s1, -r, -c1, -1.f, -c1, -r, -s1, 0.f, s1, r, c1};
    const float c = cs[x & 15], sn = cs[(x + 12) & 15];  // sin(2 pi x / 16) = cos(2 pi (x - 4) / 16)
    return SIGN < 0 ? make_float2(c, -sn) : make_float2(c, sn);
}

#ifdef FSCAN_TWQ_POW
constexpr bool kTwQPow = true;  // A/B: merged forward twiddles as powers of four table reads
#else
constexpr bool kTwQPow = false;
#endif
#ifdef FSCAN_NO_POWJ
constexpr bool kPowJ = false;  // A/B: last-stage twiddles read from the table per butterfly
#else
constexpr bool kPowJ = true;
#endif

template <int N, int R, int Ns, bool LAST, int SIGN, bool WARP, int PK, typename L, typename TW>
__device__ __forceinline__ void stage(float2 (&v)[16], int t, const L& lay, const TW& tw) {
    constexpr int T = N / 16;
    constexpr int NB = 16 / R;
    // POWJ: the last stage of a three-stage transform (span N / R > 16): butterfly
    // j of thread t has k = t + j T, so its twiddles W_N^{r (t + j T)} are the
    // thread's R - 1 table reads W_N^{r t} times the constants W_16^{r j}
    // (instead of (R - 1) NB scattered table reads: L1 wavefronts bound these
    // kernels, and the FMA pipe has room)
    constexpr bool POWJ = kPowJ && LAST && Ns > 16 && NB > 1 && (kTwPow<TW> || kTwRK<TW>);
    [[maybe_unused]] float2 tb[R];
    if constexpr (POWJ) {
        static_assert(Ns * R == N, "last stage");
#pragma unroll
        for (int r = 1; r < R; ++r) tb[r] = twiddle<SIGN>(tw, r * t);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        float2 u[R];
#pragma unroll
        for (int r = 0; r < R; ++r) u[r] = v[j + r * NB];
        const int b = t + j * T;
        const int k = b & (Ns - 1);
        if constexpr (Ns > 1) {
            constexpr int q = N / (Ns * R);  // W_{Ns R}^x = tw[x * q]
            if constexpr (POWJ) {
#pragma unroll
                for (int r = 1; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], j == 0 ? tb[r] : cmul<(PK & 2) != 0>(tb[r], w16c<SIGN>(r * j)));
            } else if constexpr (TwQInfo<TW>::kind == 1) {
                static_assert(Ns == 16 && LAST, "merged twiddles: two-stage transforms only");
                constexpr int S = TwQInfo<TW>::S;
                if (j == 0) tw.wait();
                if constexpr (kTwQPow && R == 16) {
                    // A/B: F[r][3k + q] = w^r, w = F[1][3k + q]: rows 1, 2, 4, 8 read,
                    // the other 11 powers by products (11 fewer 64-bit shared reads
                    // per transform on the L1 data pipe K4 is bound by)
                    float2 w[16];
                    w[1] = tw.at(1 * S + 3 * k);
                    w[2] = tw.at(2 * S + 3 * k);
                    w[4] = tw.at(4 * S + 3 * k);
                    w[8] = tw.at(8 * S + 3 * k);
                    w[3] = cmul(w[1], w[2]);
                    w[5] = cmul(w[4], w[1]);
                    w[6] = cmul(w[4], w[2]);
                    w[7] = cmul(w[4], w[3]);
#pragma unroll
                    for (int r = 9; r < 16; ++r) w[r] = cmul(w[8], w[r - 8]);
#pragma unroll
                    for (int r = 1; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], w[r]);
                } else {
#pragma unroll
                    for (int r = 1; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], tw.at(r * S + 3 * k));
                }
            } else if constexpr (TwQInfo<TW>::kind == 2) {
                static_assert(Ns == 16 && LAST, "merged twiddles: two-stage transforms only");
                constexpr int S = TwQInfo<TW>::S;
#pragma unroll
                for (int r = 0; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], cconj(tw.at(k * S + 3 * r)));
            } else if constexpr (Ns == 16 && kTwRK<TW>) {
                // W_{16 R}^{r k} = W_256^{(16/R) r k}
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    const float2 w = tw.rk[((16 / R) * r - 1) * 16 + k];
                    u[r] = cmul<(PK & 2) != 0>(u[r], SIGN < 0 ? w : make_float2(w.x, -w.y));
                }
            } else if constexpr (R == 16 && kTwPow<TW>) {
                // the 15 powers w^r of w = W_{16 Ns}^k from four table reads (w, w^2,
                // w^4, w^8) and 11 products: the exchanges and twiddle reads share
                // the L1 data pipe these kernels are bound by, the FMA pipe has room
                // (global tables only: K4's shared-memory table measured faster as is;
                // <= 3 rounded products per twiddle, surfaces stay ~2e-7 of the oracle)
                float2 w[16];
                w[1] = twiddle<SIGN>(tw, k * q);
                w[2] = twiddle<SIGN>(tw, 2 * k * q);
                w[4] = twiddle<SIGN>(tw, 4 * k * q);
                w[8] = twiddle<SIGN>(tw, 8 * k * q);
                w[3] = cmul<(PK & 2) != 0>(w[1], w[2]);
                w[5] = cmul<(PK & 2) != 0>(w[4], w[1]);
                w[6] = cmul<(PK & 2) != 0>(w[4], w[2]);
                w[7] = cmul<(PK & 2) != 0>(w[4], w[3]);
#pragma unroll
                for (int r = 9; r < 16; ++r) w[r] = cmul<(PK & 2) != 0>(w[8], w[r - 8]);
#pragma unroll
                for (int r = 1; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], w[r]);
            } else {
#pragma unroll
                for (int r = 1; r < R; ++r) u[r] = cmul<(PK & 2) != 0>(u[r], twiddle<SIGN>(tw, r * k * q));
            }
        }
        dft_r<R, SIGN, PK>(u);
        if constexpr (LAST) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[j + r * NB] = u[r];
        } else {
            const int base = (b / Ns) * Ns * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) lay.put(base + r * Ns, u[r]);
        }
    }
    if constexpr (!LAST) {
        exchange_sync<WARP>();
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = lay.get(t + m * T);
        exchange_sync<WARP>();
    }
}

// In-register FFT of one length-N transform (see header comment). WARP: the
// caller guarantees the transform's threads and exchange buffer live in one
// warp (row layouts with T <= 32), so the exchanges need only __syncwarp;
// otherwise every thread of the CTA must call fft_regs the same number of times.
// PK: packed fp32 (see cadd, cmul): bit 0 the butterflies' complex adds /
// subtracts, bit 1 the stage twiddle products (operands in registers), bit 2
// the radix-8 / 16 butterflies' products with compile-time constants
template <int N, int SIGN, bool WARP = false, int PK = kPkDefault, typename L, typename TW>
__device__ __forceinline__ void fft_regs(float2 (&v)[16], int t, const L& lay, const TW& tw) {
    static_assert(N >= 16 && (N & (N - 1)) == 0, "power-of-two length >= 16");
    static_assert(!WARP || N / 16 <= 32, "a warp-synchronous transform fits in one warp");
    if constexpr (N == 16) {
        stage<N, 16, 1, true, SIGN, WARP, PK>(v, t, lay, tw);
    } else if constexpr (N <= 256) {
        stage<N, 16, 1, false, SIGN, WARP, PK>(v, t, lay, tw);
        stage<N, N / 16, 16, true, SIGN, WARP, PK>(v, t, lay, tw);
    } else {
        stage<N, 16, 1, false, SIGN, WARP, PK>(v, t, lay, tw);
        stage<N, 16, 16, false, SIGN, WARP, PK>(v, t, lay, tw);
        stage<N, N / 256, 256, true, SIGN, WARP, PK>(v, t, lay, tw);
    }
}

}  // namespace fscan_fft
