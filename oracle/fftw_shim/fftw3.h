/*
 * Minimal FFTW3 API shim — TEST INFRASTRUCTURE for oracle/_ref only.
 *
 * FFTW3 is absent from this image and the reference's
 * proj/src/spectral.cpp needs exactly these declarations (spectral.cpp:22-65):
 * fftw_complex, fftw_plan, fftw_alloc_complex, fftw_free, fftw_plan_dft_2d,
 * fftw_execute, fftw_destroy_plan, FFTW_FORWARD/FFTW_BACKWARD, FFTW_ESTIMATE.
 * The transforms are the unnormalised double c2c DFTs of oracle/fft64.c.
 * This is NOT FFTW: timings of oracle/_ref are "reference CPU path with an
 * FFTW-API shim".
 */
#ifndef FSCAN_FFTW_SHIM_H
#define FSCAN_FFTW_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
