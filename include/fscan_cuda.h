/*
 * fscan_cuda.h — C ABI of the B200 (sm_100a) decoupled Fourier pose search.
 *
 * This is the drop-in boundary for the reference hot path
 *   fscan::scan_match(f, g, cfg[, mask_f, mask_g])   proj/include/fscan/matcher.hpp:72-76
 *                                                    proj/src/matcher.cpp:189-216
 * and its stage functions estimate_rotation / estimate_translation
 * (matcher.hpp:53-69). The reference has no FFI of its own (pure C++, plus a
 * pybind11 module: proj/python/module.cpp:117-136); the C++ drop-in in
 * include/fscan/ (same declarations as the reference headers) and the Python
 * package are both implemented on top of these entry points. Plain pointers
 * and sizes only; all compute happens in the sm_100a kernels of
 * paper_2203_00459_b200/csrc — there is no CPU fallback.
 *
 * Data layout: a batch of B pairs is B consecutive N x N row-major float32
 * grids per argument (f, g, mask_f, mask_g). Any grid side N in [33, 1024] is
 * supported (FSCAN_ERR_UNSUPPORTED otherwise): powers of two >= 64 take the
 * radix fast path, other sides — including the reference's own odd sizes —
 * use Bluestein DFTs in the rotation stage and a zero-embedded power-of-two
 * translation stage, in the odometry chain as well.
 *
 * Errors: every call returns an fscan_status; fscan_ctx_last_error() gives the
 * message. The C++ drop-in maps FSCAN_ERR_INVALID_ARGUMENT, _NONFINITE and
 * _MASK_RANGE to std::invalid_argument like matcher.cpp:17-37,191-193 and
 * grid.hpp:57-59,77-79, everything else to std::runtime_error.
 */
#ifndef FSCAN_CUDA_H
#define FSCAN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fscan_status {
    FSCAN_OK = 0,
    FSCAN_ERR_INVALID_ARGUMENT = 1, /* bad config / shape / pointer        */
    FSCAN_ERR_NONFINITE = 2,        /* NaN/Inf in a (masked) input grid     */
    FSCAN_ERR_MASK_RANGE = 3,       /* mask value outside [0, 1]            */
    FSCAN_ERR_UNSUPPORTED = 4,      /* valid for the reference, not here    */
    FSCAN_ERR_CUDA = 5,             /* CUDA runtime / launch failure        */
    FSCAN_ERR_NO_DEVICE = 6,        /* no usable sm_100 device              */
    FSCAN_ERR_IO = 7                /* scan file missing / malformed (fscan_io.h) */
} fscan_status;

/* fscan::MatchConfig (matcher.hpp:13-26), field for field. */
typedef struct fscan_config {
    int32_t n_theta;
    double delta_theta;
    double t_theta;
    int32_t n_xy;
    double delta_xy;
    double t_xy;
    double band_lo;
    double band_hi;
    int32_t n_radius;          /* <= 0: ceil(n_xy / 2) after finalize */
    int32_t pad_angle;         /* < 0: min(ceil(n_theta / 8), n_theta - 1) */
    int32_t softargmax_window;
    int32_t normalize_scores;  /* bool */
} fscan_config;

/* One pair's MatchResult.pose + MatchDiagnostics (matcher.hpp:32-44), plus
 * the integer hard-argmax bins behind the diagnostics. Angles in radians,
 * translations in metres (grid delta). */
typedef struct fscan_pair_result {
    double theta, tx, ty;           /* pose, theta in (-pi, pi]            */
    double theta_hard, theta_peak;  /* angular hard argmax: coord, score   */
    double xy_hard_x, xy_hard_y;    /* translation hard argmax, metres      */
    double xy_peak;                 /* translation score at that cell       */
    int32_t theta_bin;              /* row of the n_theta x 1 surface       */
    int32_t xy_row, xy_col;         /* cell of the N x N surface            */
    int32_t status;                 /* fscan_status of this pair            */
} fscan_pair_result;

typedef struct fscan_ctx fscan_ctx;

/* matcher.cpp:11-15 (finalize) and 17-37 (validate, without the odd-n rule). */
void fscan_config_defaults(fscan_config* cfg);
void fscan_config_finalize(fscan_config* cfg);
fscan_status fscan_config_validate(const fscan_config* cfg, char* msg, size_t msg_len);

/* Context = one device + one finalized config + workspace arena, tables,
 * streams. max_batch bounds the pairs per fscan_match_batch call. */
fscan_status fscan_ctx_create(int device, const fscan_config* cfg, int max_batch, fscan_ctx** out);
void fscan_ctx_destroy(fscan_ctx* ctx);
const char* fscan_ctx_last_error(const fscan_ctx* ctx);
int fscan_ctx_n(const fscan_ctx* ctx);
/* Sets the number of pairs per internal pipeline chunk (0 = automatic). */
fscan_status fscan_ctx_set_chunk(fscan_ctx* ctx, int pairs_per_chunk);

/* Batched scan_match on DEVICE pointers, asynchronous on `stream`
 * (cudaStream_t, NULL = legacy default stream). mask_f / mask_g may both be
 * NULL (unmasked overload). delta = grid metres per cell (ScanGrid.spec.delta,
 * used for the translation coordinates like matcher.cpp:162). d_out receives
 * `batch` results (device memory). d_theta_surface (batch x n_theta doubles)
 * and d_xy_surface (batch x N x N floats) are optional (NULL = not written).
 * Input validation failures (non-finite values, masks outside [0,1]) are
 * reported per pair in d_out[i].status; call fscan_check_results() or read
 * the statuses after synchronising. */
fscan_status fscan_match_batch(fscan_ctx* ctx, const float* d_f, const float* d_g,
                               const float* d_mask_f, const float* d_mask_g, int batch,
                               double delta, fscan_pair_result* d_out, double* d_theta_surface,
                               float* d_xy_surface, void* stream);

/* Config-3 hot path: raw polar sweeps (batch x n_az x n_range floats, device)
 * are resampled on the device to N x N Cartesian grids at `delta` metres per
 * cell (K0, see fscan_polar_to_cart_batch) and matched like fscan_match_batch.
 * Masks (optional) are Cartesian N x N. */
fscan_status fscan_match_batch_polar(fscan_ctx* ctx, const float* d_polar_f, const float* d_polar_g,
                                     int n_az, int n_range, double range_res, const float* d_mask_f,
                                     const float* d_mask_g, int batch, double delta,
                                     fscan_pair_result* d_out, double* d_theta_surface,
                                     float* d_xy_surface, void* stream);

/* Same on HOST pointers (pageable or pinned): host->device copies, compute and
 * device->host copy of the results, overlapped chunk by chunk; synchronous.
 * Returns the first failing pair's status (FSCAN_ERR_NONFINITE, ...). */
fscan_status fscan_match_batch_host(fscan_ctx* ctx, const float* f, const float* g,
                                    const float* mask_f, const float* mask_g, int batch,
                                    double delta, fscan_pair_result* out, double* theta_surface,
                                    float* xy_surface);

/* Stage APIs (matcher.hpp:53-69), batched, device pointers. estimate_rotation
 * writes theta (soft argmax, radians) per pair; estimate_translation takes a
 * theta per pair (device) and writes the back-rotated translation (metres). */
fscan_status fscan_estimate_rotation_batch(fscan_ctx* ctx, const float* d_f, const float* d_g,
                                           int batch, double* d_theta, double* d_theta_surface,
                                           void* stream);
fscan_status fscan_estimate_translation_batch(fscan_ctx* ctx, const float* d_f, const float* d_g,
                                              int batch, double delta, const double* d_theta,
                                              double* d_txy, float* d_xy_surface, void* stream);

/* Stage-1 intermediate for parity tests: band-passed magnitude spectrum of
 * hann(img) on the half plane u >= 0, centred rows (matcher.cpp:113-126 /
 * spectral.cpp:73-117): d_out is batch x N x W floats, W = N - N/2, element
 * [v_c][u] = |dft2(hann * img)|[v_c][N/2 + u] * band[v_c][N/2 + u]. */
fscan_status fscan_band_magnitude_batch(fscan_ctx* ctx, const float* d_img, int batch,
                                        float* d_out, void* stream);

/* K0 (config 3): raw polar sweeps (batch x n_az x n_range floats, azimuth
 * major, bin k centred at (k + 0.5) * range_res) -> batch x N x N Cartesian
 * grids at `delta` metres per cell. Spec in DESIGN.md §K0. */
fscan_status fscan_polar_to_cart_batch(const float* d_polar, int batch, int n_az, int n_range,
                                       double range_res, int n, double delta, float* d_out,
                                       void* stream);

/* Odometry over a scan sequence (the pairwise loop of proj/tools/main.cpp:124-131):
 * d_scans holds n_scans consecutive N x N grids (device), d_masks the per-scan
 * masks or NULL; pair k = scan_match(scan k, scan k+1) for k < n_scans - 1, with
 * the reference's per-pair semantics (d_out[k], optional surfaces per pair).
 * Each scan's rotation-stage spectrum and masked copy are computed once and
 * shared by its two pairs (half the K1 work of independent pairs). The host
 * side composes the trajectory (fscan/odometry.hpp: integrate of the inverse
 * poses). Asynchronous on `stream`; n_scans - 1 <= max_batch. */
fscan_status fscan_odometry_batch(fscan_ctx* ctx, const float* d_scans, const float* d_masks, int n_scans,
                                  double delta, fscan_pair_result* d_out, double* d_theta_surface,
                                  float* d_xy_surface, void* stream);

/* Brute-force correlative search (the reference's oracle, proj/src/oracle.cpp:21-67,
 * proj/include/fscan/oracle.hpp:10-23): for every candidate theta (in list
 * order) g is de-rotated by -theta and the zero-padded translation correlation
 * with f is scored; the result is the global hard argmax over (theta, row,
 * col) with ties to the earlier theta, then the lower linear index. f and g
 * are used as given (no masks, no window), like brute_force_match. */
typedef struct fscan_bf_result {
    double theta, tx, ty;   /* pose (theta normalised to (-pi, pi], t in metres) */
    double score;           /* correlation at the winning cell (OracleResult::score) */
    int32_t theta_index;    /* winning candidate */
    int32_t xy_row, xy_col; /* winning cell of the N x N lag window */
    int32_t status;         /* FSCAN_ERR_NONFINITE if the winning score is not finite */
} fscan_bf_result;

/* batch pairs (device, N x N each), n_thetas candidates from a HOST array,
 * results to device d_out[batch]. Asynchronous on `stream`. Cost: one
 * translation stage per (pair, candidate). The (pair, candidate) items run
 * through the context's chunk pipelines: a context created for fewer pairs
 * than fill them has its workspace grown once (up to ~2 GiB per pipeline, or
 * batch * n_thetas / pipelines items), which drops the cached CUDA graphs. */
fscan_status fscan_brute_force_batch(fscan_ctx* ctx, const float* d_f, const float* d_g, int batch,
                                     const double* thetas, int n_thetas, double delta,
                                     fscan_bf_result* d_out, void* stream);

/* Synchronises `stream` and scans d_out for the first non-OK status. */
fscan_status fscan_check_results(const fscan_pair_result* d_out, int batch, void* stream,
                                 int* first_bad_pair);

/* Number of kernels the last fscan_match_batch launched (for bench accounting). */
int fscan_ctx_launches_last(const fscan_ctx* ctx);
/* Spectrum columns u in [0, W) the rotation stage keeps per scan pair (the
 * columns any polar tap reads, rounded up to the column-kernel block); the row
 * kernel stores 2W - 1 columns (u < W and their mirrors). For the bench's
 * algorithmic-byte accounting. */
int fscan_ctx_rot_columns(const fscan_ctx* ctx);

/* Opt-in phase correlation (no reference code): the translation
 * stage normalises the cross-power spectrum, X / |X| (0 where X = 0), before
 * the inverse, sharpening the xy surface to a delta-like peak. The transform
 * is the GPU's length-3N/2 circular correlation (DESIGN.md §3.8 — the
 * normalisation, unlike the plain correlation, depends on that size). Off by
 * default; applies to every later call on the context. */
fscan_status fscan_ctx_set_phase_correlation(fscan_ctx* ctx, int on);

/* Profiling mode: subsequent calls run their chunks serially on one stream
 * with CUDA events around every kernel. fscan_ctx_kernel_times() synchronises
 * and returns, per kernel kind (0 rot_rows, 1 rot_cols, 2 rot_polar,
 * 3 theta_in, 4 xlat_rows, 5 xlat_cols, 6 xlat_out, 7 finalize, 8 rot_gather,
 * 9 polar_to_cart, 10 mag_unpack, 11 bf_items, 12 bf_final),
 * the summed milliseconds and launch counts of the last call. */
fscan_status fscan_ctx_set_profiling(fscan_ctx* ctx, int on);
fscan_status fscan_ctx_kernel_times(fscan_ctx* ctx, double* ms, int* launches, int n_kinds);

/* CUDA-graph replay of repeated calls (off by default). When on,
 * fscan_match_batch and fscan_odometry_batch capture their whole launch
 * sequence (every chunk, every lane) into a CUDA graph the first time they
 * see a given argument set (pointers, batch, delta, outputs) and replay it
 * with one cudaGraphLaunch on later identical calls: small batches, e.g. one
 * pair per radar sweep, stop paying ~10 launches of host overhead per call.
 * Up to 8 graphs are cached (least recently used evicted); changing the
 * context's configuration (phase correlation) or turning graphs off drops
 * them. Results are identical to the non-graph path. Profiling mode bypasses
 * graphs. */
fscan_status fscan_ctx_set_graphs(fscan_ctx* ctx, int on);
/* Graph cache statistics: captures and replays since the context was created. */
fscan_status fscan_ctx_graph_stats(const fscan_ctx* ctx, int* captures, int* replays);

#ifdef __cplusplus
}
#endif

#endif
