/* fftw3.h -- the slice of the FFTW3 API that the reference's
 * proj/src/rf/simulate.cpp uses (simulate.cpp:505-526: alloc, c2r plan,
 * execute, destroy, free), so oracle/_ref can compile that file unmodified.
 *
 * TEST INFRASTRUCTURE ONLY (oracle/Makefile).  FFTW itself is an unpinned,
 * un-vendored dependency of the reference (proj/CMakeLists.txt:16-17) absent
 * from this image; fftw_stub.c implements the published c2r definition
 * (unnormalised inverse real DFT of a Hermitian half spectrum) directly. */
#ifndef FQFG_FFTW_STUB_H
#define FQFG_FFTW_STUB_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)

fftw_complex* fftw_alloc_complex(size_t n);
double* fftw_alloc_real(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
