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

FS_HD double polar_cell(const float* polar, int n_az, int n_range, double res, int n,
                        double delta, int r, int c) {
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
    const double wa = fa - a0f;
    const long a0 = (long)a0f % n_az;
    const long a1 = (a0 + 1) % n_az;
    const double k0f = floor(fk);
    const long k0 = (long)k0f;
    const double wk = fk - k0f;
    const float* p0 = polar + (size_t)a0 * n_range;
    const float* p1 = polar + (size_t)a1 * n_range;
    const double v00 = (k0 < 0 || k0 >= n_range) ? 0.0 : (double)p0[k0];
    const double v01 = (k0 + 1 < 0 || k0 + 1 >= n_range) ? 0.0 : (double)p0[k0 + 1];
    const double v10 = (k0 < 0 || k0 >= n_range) ? 0.0 : (double)p1[k0];
    const double v11 = (k0 + 1 < 0 || k0 + 1 >= n_range) ? 0.0 : (double)p1[k0 + 1];
    return (1.0 - wa) * ((1.0 - wk) * v00 + wk * v01) + wa * ((1.0 - wk) * v10 + wk * v11);
}

}  // namespace fscan_k0
