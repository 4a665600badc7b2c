// K0 arithmetic: one Cartesian cell resampled from a raw polar sweep.
// Shared by the device kernel (kernels.cu) and the host-side generator so the
// two agree; the independent CPU restatement used for parity is
// oracle/fscan_oracle.c:fo_polar_to_cart. Spec: cell (r, c)
// sits at world x = (c - (n-1)/2) * delta, y = -(r - (n-1)/2) * delta
// (geometry.hpp:53-58 convention); azimuth bin a is centred on
// phi = 2*pi*a/n_az (CCW from +x, wrapping), range bin k on (k + 0.5) * res;
// bilinear in (azimuth, range), range taps outside [0, n_range) read zero.
#pragma once

#include <math.h>
#include <stddef.h>

#ifndef FS_HD
#ifdef __CUDACC__
#define FS_HD __host__ __device__ __forceinline__
#else
#define FS_HD inline
#endif
#endif

namespace fscan_k0 {

// Geometry of one cell (independent of the sweep values): the two azimuth
// rows, the first range bin and the bilinear weights.
struct PolarTap {
    int a0, a1;   // azimuth rows (a1 = a0 + 1 wrapped)
    int k0, pad;  // first range bin (may be outside [0, n_range))
    double wa, wk;
};

FS_HD PolarTap polar_tap(int n_az, double res, int n, double delta, int r, int c) {
    const double two_pi = 6.283185307179586;
    const int half = (n - 1) / 2;
    const double x = (c - half) * delta;
    const double y = -((r - half) * delta);
    const double rho = sqrt(x * x + y * y);
    double phi = atan2(y, x);
    if (phi < 0.0) phi += two_pi;
    const double fa = phi * (n_az / two_pi);
    const double fk = rho / res - 0.5;
    const double a0f = floor(fa);
    const long a0 = (long)a0f % n_az;
    const double k0f = floor(fk);
    PolarTap t;
    t.a0 = (int)a0;
    t.a1 = (int)((a0 + 1) % n_az);
    t.k0 = (int)(long)k0f;
    t.pad = 0;
    t.wa = fa - a0f;
    t.wk = fk - k0f;
    return t;
}

FS_HD double polar_sample(const float* polar, int n_range, const PolarTap& t) {
    const float* p0 = polar + (size_t)t.a0 * n_range;
    const float* p1 = polar + (size_t)t.a1 * n_range;
    const int k0 = t.k0;
    const bool in0 = k0 >= 0 && k0 < n_range, in1 = k0 + 1 >= 0 && k0 + 1 < n_range;
    const double v00 = in0 ? (double)p0[k0] : 0.0;
    const double v01 = in1 ? (double)p0[k0 + 1] : 0.0;
    const double v10 = in0 ? (double)p1[k0] : 0.0;
    const double v11 = in1 ? (double)p1[k0 + 1] : 0.0;
    const double wa = t.wa, wk = t.wk;
    return (1.0 - wa) * ((1.0 - wk) * v00 + wk * v01) + wa * ((1.0 - wk) * v10 + wk * v11);
}

FS_HD double polar_cell(const float* polar, int n_az, int n_range, double res, int n, double delta, int r,
                        int c) {
    return polar_sample(polar, n_range, polar_tap(n_az, res, n, delta, r, c));
}

}  // namespace fscan_k0
