/* Minimal CPU stand-in for the six FFTW3 symbols the reference's spectral
 * module uses (/root/reference/proj/src/spectral.cpp:4,136-227).
 *
 * TEST INFRASTRUCTURE ONLY: libfftw3 is absent in this image (no network), so
 * the compiled reference oracle (oracle/_ref/libhbref.so) links this shim.
 * It is a generic, unnormalised complex DFT (same sign/normalisation
 * conventions as FFTW: out[k] = sum_j in[j] * exp(sign * 2*pi*i*j*k/n)); it does
 * not know that it is being used to build the H operator.  O(n^2) per
 * transform with a precomputed twiddle table.
 */
#ifndef HB_FFTW_SHIM_H
#define HB_FFTW_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct hb_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

void* fftw_malloc(size_t n);
void fftw_free(void* p);

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex* in,
                             const int* inembed, int istride, int idist, fftw_complex* out,
                             const int* onembed, int ostride, int odist, int sign,
                             unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
