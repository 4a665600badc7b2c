// pipeline.h — device-side parameter block and kernel launchers of the
// sm_100a scan_match pipeline (kernels.cu), used by the runtime (context.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fscan_cuda.h"

namespace fscan_detail {

// One precomputed bilinear tap set of cart2pol (imageops.cpp:81-99 via
// sample_bilinear 10-26): packed = r0 | u0 << 12 | valid-tap bits << 24,
// with (r0, u0) the top-left tap in (centred row, u >= 0 column) coordinates.
struct PolarTap {
    int packed;
    float fr, fc;
    float pad_;
};

// Row pitch (float2) of the K4 -> K5 spectrum rows: 3N/4 + 1 bins rounded up
// to 8 (64-byte aligned rows). (Sizes the workspace; the layout is y_at below.)
__host__ __device__ constexpr int ypitch(int n) { return (3 * n / 4 + 1 + 7) / 8 * 8; }

// K4 -> K5 spectrum rows Y[row i][bin k'] (k' in [0, 3N/4]), stored in blocks of
// RB = y_rows(N) surface rows — exactly the rows one K5 CTA inverts — each block
// [k'][RB] float2 with the RB rows XOR-permuted per bin: K4 stores its column
// outputs straight from registers (RB consecutive rows of one bin are one
// contiguous, fully written RB * 8-byte run: no shared-memory transpose), K5
// fetches its block with one bulk copy and reads the stride-3 bins of its
// transforms conflict-free (the permutation spreads the bins a half-warp reads
// over distinct bank pairs; checked for every N by tools/bank_model.py k5y).
__host__ __device__ constexpr int y_rows(int n) { return 4096 / n < n ? 4096 / n : n; }
__host__ __device__ constexpr int y_swz(int rb, int k) {
    return (rb / 4) * ((k >> (rb >= 16 ? 0 : (rb == 8 ? 1 : 2))) & 3);
}
// float2 offset of Y[i][k] inside one pair's rows
template <int N>
__host__ __device__ constexpr int y_at(int i, int k) {
    constexpr int RB = y_rows(N), H1 = 3 * N / 4 + 1;
    return ((i / RB) * H1 + k) * RB + ((i % RB) ^ y_swz(RB, k));
}

// Per-pair state handed from the angular stage to the translation stage.
struct RotState {
    double theta;      // soft-argmax theta (radians, not wrapped)
    double st, ct;     // sin(-theta), cos(-theta) for rotate_bilinear(g, -theta)
    double peak;       // theta surface at the hard argmax
    double hard;       // coordinate of the hard argmax
    int bin;           // hard argmax row
    int identity;      // -theta == 0.0: rotate_bilinear returns g unchanged
};

struct Partial {
    float val;
    int idx;
};

struct Params {
    int n;        // grid side N (power of two)
    int batch;    // pairs in this launch
    // inputs (device)
    const float* f;
    const float* g;
    const float* mf;  // nullable
    const float* mg;
    // workspace
    float* ft;     // masked f  [batch][N][N]
    float* gt;     // masked g
    float2* zbuf;  // K1a->K1b spectra [batch][N][N]; reused as K4->K5 rows [batch][N][3N/4+1]
    float* mag;    // (|F|,|G|) band-passed half planes, tiled [batch][N/16][N][8] float2; reused as surface
    float2* fgt;   // row spectra of f, g_rot (length 3N/2), transposed [batch][F, G plane][3N/4+1][N]
    float* surf;   // translation surface [batch][N][N]
    Partial* part; // K5 per-block argmax [batch][N / rows_per_block]
    RotState* rot; // [batch]
    double* prof;  // K2a radial-sum profiles [batch][2][n_theta]
    double* theta_ws;  // K2b split over several CTAs per pair (small batches): scores [batch][n_theta]
    int* polar_cnt;    // split K2b: finished CTAs per pair [batch], zero between launches (nullptr: separate fin kernel)
    int* flags;    // [batch] (chain mode: [n_scans]) bit0 non-finite, bit1 mask out of [0,1]
    // tables
    const float2* tw_n;   // exp(-2 pi i k / N), k < N
    const float2* tw_k;   // exp(-2 pi i k / K), K = N/2
    const float2* tw_k2;  // exp(-2 pi i k / (K/2))
    const float2* tw_m;   // exp(-2 pi i k / M), M = 3N/2
    const float2* tw_rk;  // exp(-2 pi i r k / 256) at (r-1)*16 + k, r < 16, k < 16
    const float2* tw_k4;  // K4 merged twiddles W_M^{a j} at a*48 + j, a < 16, j < 48 (fft.cuh SmemTwQF)
    const float* hann;    // N
    const int2* band;     // per centred row: [u_lo, u_hi] in band (empty: lo > hi)
    const PolarTap* taps; // [n_live][n_theta] (radius-major)
    int n_live;
    int zcols;            // K1b computes columns u < zcols (multiple of 8); K1a stores only those and their mirrors
    // config
    int n_theta, pad, L, C;
    double delta_theta, t_theta, t_xy, delta;
    int window, normalize;
    // outputs
    fscan_pair_result* out;   // nullable for stage calls
    double* theta_surf;       // nullable
    float* xy_surf;           // nullable (else surf is workspace)
    double* theta_only;       // stage API: theta per pair (nullable)
    double* txy_only;         // stage API: (tx, ty) per pair (nullable)
    const double* theta_in;   // stage API: theta per pair for translation-only runs
    float* mag_out;           // stage API: band magnitude, [batch][N][N/2] (nullable)
    // translation items: item i of this launch is global item item_base + i; it
    // reads the masked scans of pair (item_base + i) / src_div (1 for matching;
    // the candidate count for the brute-force search) and, with theta_mod > 0,
    // theta_in[(item_base + i) % theta_mod]
    int item_base, src_div, theta_mod;
    int skip_surface;         // K5 keeps only the block argmaxes (brute-force search)
    int phase;                // opt-in phase correlation (K4 normalises the cross-power)
    // chain mode (odometry): pair k registers scan k against scan k+1 of one
    // sequence f (masks mf); K1a/K1b run once per two scans (n_scans of them in
    // this launch), the masked scans go to ft[scan], the magnitude planes and
    // the flags are one per scan
    int chain, n_scans;
    Partial* bf_items;        // brute force: per global item hard argmax (nullable)
    // Grid sides that are not powers of two (the reference's odd sizes), see
    // DESIGN.md §3.9. The rotation stage runs at N = n with Bluestein DFTs of
    // length bs_L; the translation stage runs at np (a power of two >= N + 1)
    // on zero-embedded scans: rotation centre c0, valid grid n, lag window at
    // offset win_off in the np x np surface. pow2: n == np, c0 = (n-1)/2, off 0.
    int np;
    float c0;
    int win_off;
    int embed;                // 1: translation stage embedded (n < np)
    int pdl;                  // 1: pipeline kernels launched with programmatic stream serialisation
    int nw;                   // half-plane width W = n - n/2 (u in [0, W))
    long long mag_plane;      // float2 per (|F|,|G|) tile set: n * 8 * ceil(W / 8)
    int bs_L;                 // Bluestein transform length (0: pow2 fast path)
    const float2* bs_chirp;   // exp(-i pi k^2 / n), k < n
    const float2* bs_kern;    // FFT_L of the chirp kernel, / L
    const float2* tw_L;       // exp(-2 pi i k / L), k < L
    // K3's de-rotation gather through the texture path (tld4: the 2x2 taps of a
    // cell in one fetch): a pitch-2D texture over the lane's masked-g buffer,
    // rows pair * np + r; used only while gt == gtex_base (0: plain loads)
    unsigned long long gtex;
    const float* gtex_base;
};

// Launch the stages; each returns cudaGetLastError() of its launch.
cudaError_t launch_rot_rows(const Params& p, cudaStream_t s);        // K1a
cudaError_t launch_rot_cols(const Params& p, cudaStream_t s);        // K1b
cudaError_t launch_rot_gather(const Params& p, cudaStream_t s);      // K2a
cudaError_t launch_rot_polar(const Params& p, cudaStream_t s);       // K2b
cudaError_t launch_theta_in(const Params& p, cudaStream_t s);        // stage API: theta from caller
cudaError_t launch_xlat_rows(const Params& p, cudaStream_t s);       // K3
cudaError_t launch_xlat_cols(const Params& p, cudaStream_t s);       // K4
cudaError_t launch_xlat_out(const Params& p, cudaStream_t s);        // K5
cudaError_t launch_xlat_win(const Params& p, cudaStream_t s);        // K5 window rows (two-pass form)
bool xlat_win_pass(const Params& p);  // K5 runs as block maxima + window rows
cudaError_t launch_finalize(const Params& p, cudaStream_t s);        // K6
cudaError_t launch_mag_unpack(const Params& p, cudaStream_t s);      // stage API helper
cudaError_t launch_bf_items(const Params& p, cudaStream_t s);        // brute force: item argmax
// brute force: winner per pair (np: surface pitch, off: lag-window offset, §3.9)
cudaError_t launch_bf_final(const Partial* items, const double* thetas, int n_thetas, int batch, int n, int np,
                            int off, double delta, fscan_bf_result* out, cudaStream_t s);
cudaError_t launch_embed(const float* src, int count, int n, int np, float* dst, cudaStream_t s);
cudaError_t launch_rot_rows_bs(const Params& p, cudaStream_t s);     // K1a, Bluestein (any n)
cudaError_t launch_rot_cols_bs(const Params& p, cudaStream_t s);     // K1b, Bluestein (any n)
// K0: one or two sweep batches (d_polar1 nullable) -> Cartesian grids through
// a per-geometry tap table `tab` (polar_tap_bytes(n), built by
// launch_polar_taps; nullptr: a temporary one is built for the call)
size_t polar_tap_bytes(int n);
cudaError_t launch_polar_taps(int n_az, double range_res, int n, double delta, void* tab, cudaStream_t stream);
cudaError_t launch_polar_to_cart(const float* d_polar0, const float* d_polar1, int batch, int n_az,
                                 int n_range, double range_res, int n, double delta, float* d_out0,
                                 float* d_out1, cudaStream_t stream, const void* tab = nullptr);
int rows_per_block_out(int n);  // K5 rows per CTA (partials per pair = n / this)

}  // namespace fscan_detail
