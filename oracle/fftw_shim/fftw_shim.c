#define _POSIX_C_SOURCE 200112L
/* FFTW-API shim over oracle/fft64.c — TEST INFRASTRUCTURE (see fftw3.h). */
#include "fftw3.h"

#include <stdlib.h>
#include <string.h>

#include "../fft64.h"

struct fftw_plan_s {
    int rows, cols, sign;
    fftw_complex* in;
    fftw_complex* out;
    fft64_plan* prow; /* length cols */
    fft64_plan* pcol; /* length rows */
    double* colbuf;
};

fftw_complex* fftw_alloc_complex(size_t n) {
    void* p = NULL;
    if (posix_memalign(&p, 64, (n ? n : 1) * sizeof(fftw_complex)) != 0) return NULL;
    return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags) {
    (void)flags;
    if (n0 < 1 || n1 < 1 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return NULL;
    struct fftw_plan_s* p = (struct fftw_plan_s*)calloc(1, sizeof(*p));
    if (!p) return NULL;
    p->rows = n0;
    p->cols = n1;
    p->sign = sign;
    p->in = in;
    p->out = out;
    p->prow = fft64_plan_1d(n1);
    p->pcol = fft64_plan_1d(n0);
    p->colbuf = (double*)malloc(sizeof(double) * 2 * (size_t)n0);
    if (!p->prow || !p->pcol || !p->colbuf) {
        fftw_destroy_plan(p);
        return NULL;
    }
    return p;
}

void fftw_execute(const fftw_plan p) {
    const int rows = p->rows, cols = p->cols;
    double* x = (double*)p->out;
    if (p->in != p->out) memcpy(x, p->in, sizeof(fftw_complex) * (size_t)rows * cols);
    for (int r = 0; r < rows; ++r) fft64_exec_1d(p->prow, x + 2 * (size_t)r * cols, p->sign);
    double* col = p->colbuf;
    for (int c = 0; c < cols; ++c) {
        for (int r = 0; r < rows; ++r) {
            col[2 * r] = x[2 * ((size_t)r * cols + c)];
            col[2 * r + 1] = x[2 * ((size_t)r * cols + c) + 1];
        }
        fft64_exec_1d(p->pcol, col, p->sign);
        for (int r = 0; r < rows; ++r) {
            x[2 * ((size_t)r * cols + c)] = col[2 * r];
            x[2 * ((size_t)r * cols + c) + 1] = col[2 * r + 1];
        }
    }
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    fft64_destroy(p->prow);
    fft64_destroy(p->pcol);
    free(p->colbuf);
    free(p);
}
