/*
 * fft64 — double-precision complex DFT used ONLY by the parity oracle.
 *
 * TEST INFRASTRUCTURE. Nothing on the product path links this file; it backs
 * (a) the C restatement in oracle/fscan_oracle.c and (b) the FFTW-API shim
 * that lets the reference's own spectral.cpp compile into oracle/_ref/.
 *
 * It restates the published algorithm the reference delegates to FFTW3
 * (un-vendored, version unpinned: proj/CMakeLists.txt:15): an unnormalised
 * complex DFT  X[k] = sum_j x[j] * exp(sign * 2*pi*i * j*k / n), sign = -1 for
 * forward and +1 for backward (FFTW_FORWARD / FFTW_BACKWARD convention used at
 * proj/src/spectral.cpp:49-52). Sizes whose prime factors are all <= 13 use a
 * mixed-radix Cooley-Tukey recursion; any other size uses Bluestein's chirp-z
 * identity over a power-of-two convolution, so every n is exact to ~1e-15.
 *
 * Data are interleaved (re, im) doubles, the memory layout of fftw_complex.
 */
#ifndef FSCAN_ORACLE_FFT64_H
#define FSCAN_ORACLE_FFT64_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fft64_plan fft64_plan;

/* Plan for a 1-D transform of length n (n >= 1). Returns NULL on failure. */
fft64_plan* fft64_plan_1d(int n);
void fft64_destroy(fft64_plan* p);

/* In-place 1-D transform of `data` (2*n doubles), sign = -1 or +1. */
void fft64_exec_1d(const fft64_plan* p, double* data, int sign);

/* In-place row-major 2-D transform of a rows x cols complex array. */
void fft64_exec_2d(int rows, int cols, double* data, int sign);

#ifdef __cplusplus
}
#endif

#endif
