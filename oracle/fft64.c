/*
 * fft64 — double-precision complex DFT for the parity oracle (TEST
 * INFRASTRUCTURE ONLY; see fft64.h). Restates the unnormalised DFT that the
 * reference obtains from FFTW3 (proj/src/spectral.cpp:22-65): mixed-radix
 * Cooley-Tukey (decimation in time, radices 4,2,3,5,7,11,13) with one exact
 * twiddle table per plan, and Bluestein's chirp-z algorithm for lengths with a
 * larger prime factor (e.g. the 109 in the rotation-stage sizes 218/436/872).
 */
#include "fft64.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

struct fft64_plan {
    int n;
    int nfac;
    int fac[64];
    cplx* tw; /* tw[x] = exp(-2*pi*i*x/n) */
    /* Bluestein */
    int blue;
    int m;
    cplx* chirp;     /* exp(-i*pi*(j^2 mod 2n)/n), j < n */
    cplx* kern_fwd;  /* FFT_m of the forward convolution kernel */
    cplx* kern_bwd;  /* FFT_m of the backward convolution kernel */
    fft64_plan* sub; /* power-of-two plan of length m */
};

static const double kTwoPi = 6.283185307179586476925286766559;
static const double kPiD = 3.14159265358979323846264338327950288;

static int factorize(int n, int* fac) {
    int k = 0;
    while (n % 4 == 0) { fac[k++] = 4; n /= 4; }
    static const int primes[] = {2, 3, 5, 7, 11, 13};
    for (int i = 0; i < 6; ++i)
        while (n % primes[i] == 0) { fac[k++] = primes[i]; n /= primes[i]; }
    return n == 1 ? k : -1;
}

fft64_plan* fft64_plan_1d(int n) {
    if (n < 1) return NULL;
    fft64_plan* p = (fft64_plan*)calloc(1, sizeof(fft64_plan));
    if (!p) return NULL;
    p->n = n;
    p->nfac = factorize(n, p->fac);
    if (p->nfac >= 0) {
        p->tw = (cplx*)malloc(sizeof(cplx) * (size_t)n);
        for (int x = 0; x < n; ++x) {
            const double a = -kTwoPi * (double)x / (double)n;
            p->tw[x] = cos(a) + I * sin(a);
        }
        return p;
    }
    /* Bluestein: X[k] = c[k] * sum_j (x[j] c[j]) conj(c[k-j]), c[j] = w^(j^2/2) */
    p->blue = 1;
    int m = 1;
    while (m < 2 * n - 1) m <<= 1;
    p->m = m;
    p->sub = fft64_plan_1d(m);
    p->chirp = (cplx*)malloc(sizeof(cplx) * (size_t)n);
    p->kern_fwd = (cplx*)calloc((size_t)m, sizeof(cplx));
    p->kern_bwd = (cplx*)calloc((size_t)m, sizeof(cplx));
    for (int j = 0; j < n; ++j) {
        const long long q = ((long long)j * j) % (2LL * n);
        const double a = -kPiD * (double)q / (double)n;
        p->chirp[j] = cos(a) + I * sin(a);
    }
    for (int j = 0; j < n; ++j) {
        p->kern_fwd[j] = conj(p->chirp[j]);
        p->kern_bwd[j] = p->chirp[j];
        if (j > 0) {
            p->kern_fwd[m - j] = conj(p->chirp[j]);
            p->kern_bwd[m - j] = p->chirp[j];
        }
    }
    fft64_exec_1d(p->sub, (double*)p->kern_fwd, -1);
    fft64_exec_1d(p->sub, (double*)p->kern_bwd, -1);
    return p;
}

void fft64_destroy(fft64_plan* p) {
    if (!p) return;
    free(p->tw);
    free(p->chirp);
    free(p->kern_fwd);
    free(p->kern_bwd);
    fft64_destroy(p->sub);
    free(p);
}

/* DFT of the n samples in[0], in[s], in[2s], ... into out[0..n). */
static void ct_rec(cplx* out, const cplx* in, int n, int s, const int* fac,
                   const cplx* tw, int ntot, int sign) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    const int p = fac[0];
    const int m = n / p;
    for (int j = 0; j < p; ++j) ct_rec(out + j * m, in + j * s, m, s * p, fac + 1, tw, ntot, sign);
    const int tstride = ntot / n; /* W_n^x = tw[x * tstride] */
    const int pstride = ntot / p; /* W_p^x = tw[x * pstride] */
    cplx y[16];
    for (int k = 0; k < m; ++k) {
        for (int j = 0; j < p; ++j) {
            cplx w = tw[(size_t)j * k * tstride];
            if (sign > 0) w = conj(w);
            y[j] = out[j * m + k] * w;
        }
        if (p == 2) {
            out[k] = y[0] + y[1];
            out[m + k] = y[0] - y[1];
        } else if (p == 4) {
            const cplx a = y[0] + y[2], b = y[0] - y[2];
            const cplx c = y[1] + y[3];
            cplx d = y[1] - y[3];
            d = (sign < 0) ? (-I * d) : (I * d);
            out[k] = a + c;
            out[m + k] = b + d;
            out[2 * m + k] = a - c;
            out[3 * m + k] = b - d;
        } else {
            for (int q = 0; q < p; ++q) {
                cplx acc = 0.0;
                for (int j = 0; j < p; ++j) {
                    cplx w = tw[(size_t)((j * q) % p) * pstride];
                    if (sign > 0) w = conj(w);
                    acc += y[j] * w;
                }
                out[q * m + k] = acc;
            }
        }
    }
}

void fft64_exec_1d(const fft64_plan* p, double* data, int sign) {
    const int n = p->n;
    cplx* x = (cplx*)data;
    if (!p->blue) {
        cplx* tmp = (cplx*)malloc(sizeof(cplx) * (size_t)n);
        ct_rec(tmp, x, n, 1, p->fac, p->tw, n, sign);
        memcpy(x, tmp, sizeof(cplx) * (size_t)n);
        free(tmp);
        return;
    }
    const int m = p->m;
    cplx* a = (cplx*)calloc((size_t)m, sizeof(cplx));
    for (int j = 0; j < n; ++j) {
        const cplx c = (sign < 0) ? p->chirp[j] : conj(p->chirp[j]);
        a[j] = x[j] * c;
    }
    fft64_exec_1d(p->sub, (double*)a, -1);
    const cplx* kern = (sign < 0) ? p->kern_fwd : p->kern_bwd;
    for (int j = 0; j < m; ++j) a[j] *= kern[j];
    fft64_exec_1d(p->sub, (double*)a, +1);
    const double inv = 1.0 / (double)m;
    for (int k = 0; k < n; ++k) {
        const cplx c = (sign < 0) ? p->chirp[k] : conj(p->chirp[k]);
        x[k] = a[k] * inv * c;
    }
    free(a);
}

void fft64_exec_2d(int rows, int cols, double* data, int sign) {
    fft64_plan* pr = fft64_plan_1d(cols);
    fft64_plan* pc = (rows == cols) ? pr : fft64_plan_1d(rows);
    cplx* x = (cplx*)data;
    for (int r = 0; r < rows; ++r) fft64_exec_1d(pr, (double*)(x + (size_t)r * cols), sign);
    cplx* col = (cplx*)malloc(sizeof(cplx) * (size_t)rows);
    for (int c = 0; c < cols; ++c) {
        for (int r = 0; r < rows; ++r) col[r] = x[(size_t)r * cols + c];
        fft64_exec_1d(pc, (double*)col, sign);
        for (int r = 0; r < rows; ++r) x[(size_t)r * cols + c] = col[r];
    }
    free(col);
    if (pc != pr) fft64_destroy(pc);
    fft64_destroy(pr);
}
