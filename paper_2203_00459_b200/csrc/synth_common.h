// Shared host/device pieces of the synthetic scan generator (fscan_synth.h).
// Harness code: produces inputs for tests and the bench, never part of a
// timed region.
#pragma once

#include <math.h>
#include <stdint.h>

#include "fscan_synth.h"
#include "polar.h"

namespace fsynth {

constexpr double kPi = 3.141592653589793;

// splitmix64 finaliser (the core of proj/include/fscan/rng.hpp:17-23).
FS_HD uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Stream key for (seed, pair, scan, purpose) — the Rng::mix derivation of
// rng.hpp:47-50 applied twice.
FS_HD uint64_t stream_key(uint64_t seed, uint64_t pair, uint64_t scan, uint64_t purpose) {
    uint64_t k = mix64(seed ^ (0xD1B54A32D192ED03ull * (pair + 1)));
    k = mix64(k ^ (0xA24BAED4963EE407ull * (scan + 1)));
    return mix64(k ^ (0x9FB21C651E98DF25ull * (purpose + 1)));
}

// Counter-based uniform in [0, 1).
FS_HD double u01(uint64_t key, uint64_t i) {
    return (double)(mix64(key ^ mix64(i)) >> 11) * 0x1.0p-53;
}

// Rayleigh(scale) = scale * sqrt(-2 ln(1 - U)).
FS_HD double rayleigh(uint64_t key, uint64_t i, double scale) {
    return scale * sqrt(-2.0 * log(1.0 - u01(key, i)));
}

// Box-Muller standard normal from two counter draws.
FS_HD double normal(uint64_t key, uint64_t i) {
    const double u1 = 1.0 - u01(key, 2 * i);
    const double u2 = u01(key, 2 * i + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

// Sequential splitmix64 stream for per-pair scene parameters (rng.hpp:13-29).
struct Seq {
    uint64_t s;
    FS_HD explicit Seq(uint64_t seed) : s(seed) {}
    FS_HD uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    FS_HD double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    FS_HD double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

// One scene object: a Gaussian-profile segment; reflectors are zero-length
// segments. Coordinates in metres (world frame, x right, y up).
struct Object {
    double x0, y0, x1, y1;
    double inv2s2;  // 1 / (2 sigma^2)
    double cut2;    // contributions beyond (5 sigma)^2 are dropped
    double amp;
};

FS_HD double object_value(const Object& o, double x, double y) {
    const double vx = o.x1 - o.x0, vy = o.y1 - o.y0;
    const double l2 = vx * vx + vy * vy;
    double t = 0.0;
    if (l2 > 0.0) {
        t = ((x - o.x0) * vx + (y - o.y0) * vy) / l2;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double dx = x - (o.x0 + t * vx), dy = y - (o.y0 + t * vy);
    const double d2 = dx * dx + dy * dy;
    return d2 <= o.cut2 ? o.amp * exp(-d2 * o.inv2s2) : 0.0;
}

// World position of cell (r, c): GridSpec convention, integer (n-1)/2
// (proj/include/fscan/geometry.hpp:53-58).
FS_HD void cell_world(int n, double delta, int r, int c, double* x, double* y) {
    const int half = (n - 1) / 2;
    *x = (c - half) * delta;
    *y = -((r - half) * delta);
}

FS_HD double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

}  // namespace fsynth
