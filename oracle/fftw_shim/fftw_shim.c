#define _POSIX_C_SOURCE 200112L
/* Generic naive complex DFT implementing the FFTW3 subset declared in
 * fftw3.h.  Test infrastructure for the compiled reference oracle only.
 * Supported plan shapes: rank 1, unit stride, contiguous batches
 * (idist = odist = n), which is all the reference requests
 * (/root/reference/proj/src/spectral.cpp:157-163).
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct hb_fftw_plan_s {
    int n;
    int howmany;
    int istride, idist, ostride, odist;
    int sign;
    double* tw; /* 2*n: cos, sin of sign*2*pi*m/n */
};

void* fftw_malloc(size_t n) {
    void* p = NULL;
    if (posix_memalign(&p, 64, n ? n : 1) != 0)
        return NULL;
    return p;
}

void fftw_free(void* p) { free(p); }

static fftw_plan make_plan(int n, int howmany, int istride, int idist, int ostride, int odist,
                           int sign) {
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->n = n;
    p->howmany = howmany;
    p->istride = istride;
    p->idist = idist;
    p->ostride = ostride;
    p->odist = odist;
    p->sign = sign;
    p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    const double two_pi = 6.283185307179586476925286766559;
    for (int m = 0; m < n; ++m) {
        const double ph = (double)sign * two_pi * (double)m / (double)n;
        p->tw[2 * m] = cos(ph);
        p->tw[2 * m + 1] = sin(ph);
    }
    return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    return make_plan(n, 1, 1, n, 1, n, sign);
}

fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex* in,
                             const int* inembed, int istride, int idist, fftw_complex* out,
                             const int* onembed, int ostride, int odist, int sign,
                             unsigned flags) {
    (void)in;
    (void)out;
    (void)inembed;
    (void)onembed;
    (void)flags;
    if (rank != 1)
        return NULL;
    return make_plan(n[0], howmany, istride, idist, ostride, odist, sign);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n = p->n;
    double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    for (int b = 0; b < p->howmany; ++b) {
        const fftw_complex* src = in + (size_t)b * (size_t)p->idist;
        fftw_complex* dst = out + (size_t)b * (size_t)p->odist;
        for (int k = 0; k < n; ++k) {
            double re = 0.0, im = 0.0;
            int m = 0; /* (j*k) mod n, advanced incrementally */
            for (int j = 0; j < n; ++j) {
                const double c = p->tw[2 * m], s = p->tw[2 * m + 1];
                const double xr = src[(size_t)j * (size_t)p->istride][0];
                const double xi = src[(size_t)j * (size_t)p->istride][1];
                re += xr * c - xi * s;
                im += xr * s + xi * c;
                m += k;
                if (m >= n)
                    m -= n;
            }
            tmp[2 * k] = re;
            tmp[2 * k + 1] = im;
        }
        for (int k = 0; k < n; ++k) {
            dst[(size_t)k * (size_t)p->ostride][0] = tmp[2 * k];
            dst[(size_t)k * (size_t)p->ostride][1] = tmp[2 * k + 1];
        }
    }
    free(tmp);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p)
        return;
    free(p->tw);
    free(p);
}
