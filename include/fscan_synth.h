/*
 * fscan_synth.h — seeded synthetic scan-pair generator for the BASELINE
 * configurations (BASELINE.json "configs").
 *
 * The reference's own generator (proj/src/synth.cpp: Gaussian blobs + Gaussian
 * speckle) does not produce the BASELINE workloads, so this is a
 * new generator. Its random-stream design follows proj/include/fscan/rng.hpp:
 * splitmix64 with per-pair streams derived from (seed, pair index), so pair k
 * is the same pair whatever the batch size, shard or GPU count. Per-pixel
 * noise is counter-based (hash of seed, pair, scan, pixel), which lets the host
 * and the device renderers produce the same field up to libm rounding.
 *
 * Pose convention (proj/include/fscan/matcher.hpp:71, synth.cpp:99-109):
 * scan A is the scene at the identity, scan B the scene after pose p, so that
 * f(x) ~= g(apply(p, x)) and the matcher's target is exactly p.
 */
#ifndef FSCAN_SYNTH_H
#define FSCAN_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fscan_synth_spec {
    int polar;            /* 0: render Cartesian directly; 1: render raw polar sweeps */
    int n;                /* Cartesian side (cells) */
    double delta;         /* metres per cell */
    int n_reflectors;     /* Gaussian point reflectors per scene */
    int n_segments;       /* Gaussian line segments per scene */
    double sigma_lo_px;   /* reflector sigma ~ U(lo, hi) cells */
    double sigma_hi_px;
    double seg_sigma_px;  /* segment cross-section sigma, cells */
    double extent_frac;   /* objects lie in the central extent_frac of the grid */
    double theta_max;     /* theta ~ U(-theta_max, theta_max), radians */
    double t_max;         /* t ~ U(-t_max, t_max) per axis, metres */
    double speckle;       /* Rayleigh scale of the additive speckle */
    int masks;            /* 0: all-ones masks; 1: box5x5(sigmoid(N(0, mask_sigma))) */
    double mask_sigma;
    /* polar sweeps (polar = 1) */
    int n_az;
    int n_range;
    double range_res;     /* metres per range bin */
    double att_r0;        /* returns scale by (att_r0 / max(rho, att_r0))^2 */
    uint64_t seed;
} fscan_synth_spec;

/* Config presets 1..5 of BASELINE.json. Returns 0, or -1 for an unknown id. */
int fscan_synth_preset(int config_id, fscan_synth_spec* out);

/* Host rendering of pairs [first, first + count). f/g/mf/mg are count*n*n
 * floats (mf/mg may be NULL); truth (may be NULL) receives theta, tx, ty per
 * pair. Polar specs are resampled to Cartesian on the CPU (same spec as the
 * device K0 kernel). threads <= 0 uses every hardware thread. */
int fscan_synth_pairs_host(const fscan_synth_spec* spec, int first, int count, float* f,
                           float* g, float* mf, float* mg, double* truth, int threads);

/* Host rendering of raw polar sweeps (polar specs only): pf/pg are
 * count * n_az * n_range floats. */
int fscan_synth_polar_host(const fscan_synth_spec* spec, int first, int count, float* pf,
                           float* pg, double* truth, int threads);

/* Device rendering of Cartesian pairs into device buffers (polar specs are
 * rendered as sweeps and converted by the product K0 kernel). */
int fscan_synth_pairs_device(const fscan_synth_spec* spec, int first, int count, float* d_f,
                             float* d_g, float* d_mf, float* d_mg, double* truth, void* stream);

/* Device rendering of a scan SEQUENCE (odometry workloads): `count` scans of
 * the scene of pair `seq`, scan k seen after pose P_k (P_0 = identity, P_k the
 * pose pair seq + k would draw: independent and bounded, so consecutive scans
 * differ like generator pairs, up to twice the pose range). d_scans (and
 * d_masks, per scan, may be NULL) hold count * n * n floats; truth (host, may
 * be NULL) receives P_k as theta, tx, ty per scan; the relative pose of
 * (scan k, scan k+1) in the matcher's convention is P_{k+1} o inverse(P_k). */
int fscan_synth_sequence_device(const fscan_synth_spec* spec, int seq, int count, float* d_scans,
                                float* d_masks, double* truth, void* stream);

/* Device rendering of raw polar sweeps into device buffers. */
int fscan_synth_polar_device(const fscan_synth_spec* spec, int first, int count, float* d_pf,
                             float* d_pg, double* truth, void* stream);

#ifdef __cplusplus
}
#endif

#endif
