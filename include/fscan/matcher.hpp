// fscan/matcher.hpp — the hot-path API of the reference
// (proj/include/fscan/matcher.hpp:13-76), implemented on the B200 through the
// C ABI in fscan_cuda.h. Same declarations, argument meaning and exceptions:
// std::invalid_argument for bad configs, mismatched grids, non-finite inputs
// and masks outside [0, 1]; std::runtime_error for device failures.
// Added: scan_match_batch for many pairs resident in device memory.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "fscan/types.hpp"

namespace fscan {

struct MatchConfig {
    int n_theta = 733;
    double delta_theta = kPi / 733.0;
    double t_theta = 2.0;      // angular softmax gain
    int n_xy = 255;
    double delta_xy = 0.4;
    double t_xy = 1.0;         // translation softmax gain
    double band_lo = 0.03;     // annulus, fractions of Nyquist
    double band_hi = 0.75;
    int n_radius = 128;        // <= 0: ceil(n_xy / 2)
    int pad_angle = 92;        // < 0: ceil(n_theta / 8), capped at n_theta - 1
    int softargmax_window = 16;
    bool normalize_scores = true;
};

void finalize(MatchConfig& cfg);
void validate(const MatchConfig& cfg);

struct MatchDiagnostics {
    double theta_peak = 0.0;
    double theta_hard = 0.0;
    double xy_peak = 0.0;
    Vec2 xy_hard{0.0, 0.0};
};

struct MatchResult {
    Pose2D pose;
    CorrelationSurface theta_surface;  // n_theta x 1
    CorrelationSurface xy_surface;     // n_xy x n_xy, rows t_y', cols t_x'
    MatchDiagnostics diagnostics;
};

std::pair<double, double> soft_argmax(const CorrelationSurface& s, double gain, int window,
                                      bool normalize = true);

std::pair<double, CorrelationSurface> estimate_rotation(const ScanGrid& f, const ScanGrid& g,
                                                        const MatchConfig& cfg);

std::pair<Vec2, CorrelationSurface> estimate_translation(const ScanGrid& f, const ScanGrid& g,
                                                         double theta, const MatchConfig& cfg);

MatchResult scan_match(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg);
MatchResult scan_match(const ScanGrid& f, const ScanGrid& g, const MatchConfig& cfg,
                       const MaskGrid& mask_f, const MaskGrid& mask_g);

// Batched extension: `batch` pairs of n_xy x n_xy float32 grids already on
// device `device` (masks may be null), results written to host `poses`
// (and `diags` if non-null). Synchronous; throws like scan_match.
struct PairDiagnostics {
    MatchDiagnostics diag;
    int theta_bin = 0;
    int xy_row = 0;
    int xy_col = 0;
};
void scan_match_batch(const float* d_f, const float* d_g, const float* d_mask_f,
                      const float* d_mask_g, int batch, double delta, const MatchConfig& cfg,
                      std::vector<Pose2D>& poses, std::vector<PairDiagnostics>* diags = nullptr,
                      int device = 0);

}  // namespace fscan
