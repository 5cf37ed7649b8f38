/* fftw_stub.c -- FFTW3's fftw_plan_dft_c2r_1d semantics, by definition.
 *
 * TEST INFRASTRUCTURE ONLY: lets oracle/_ref compile the reference's
 * rf/simulate.cpp (see fftw3.h).  For a plan of size n over the half
 * spectrum in[0 .. n/2]:
 *
 *   out[m] = Re in[0] + 2 sum_{k=1}^{ceil(n/2)-1} Re(in[k] e^{+2 pi i k m / n})
 *            + (n even) Re in[n/2] (-1)^m
 *
 * unnormalised, imaginary parts of in[0] and in[n/2] ignored -- FFTW's
 * documented c2r transform.  O(n x nonzero bins), FP64, twiddles from the
 * exactly reduced index (k m mod n) so every angle is computed once to
 * within an ulp; the simulator's spectra occupy only the passband bins. */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct fftw_plan_s {
  int n;
  fftw_complex* in;
  double* out;
  double* cs; /* cos(2 pi j / n), j < n */
  double* sn;
};

fftw_complex* fftw_alloc_complex(size_t n) { return (fftw_complex*)malloc(n * sizeof(fftw_complex)); }

double* fftw_alloc_real(size_t n) { return (double*)malloc(n * sizeof(double)); }

void fftw_free(void* p) { free(p); }

fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags) {
  (void)flags;
  if (n < 1 || !in || !out) return NULL;
  fftw_plan p = (fftw_plan)calloc(1, sizeof *p);
  if (!p) return NULL;
  p->n = n;
  p->in = in;
  p->out = out;
  p->cs = (double*)malloc((size_t)n * sizeof(double));
  p->sn = (double*)malloc((size_t)n * sizeof(double));
  const double two_pi = 6.283185307179586476925286766559;
  for (int j = 0; j < n; ++j) {
    p->cs[j] = cos(two_pi * (double)j / (double)n);
    p->sn[j] = sin(two_pi * (double)j / (double)n);
  }
  return p;
}

void fftw_execute(const fftw_plan p) {
  const int n = p->n, half = n / 2;
  const int kmax = (n % 2 == 0) ? half - 1 : half; /* bins with a conjugate twin */
  /* the nonzero interior bins */
  int* nz = (int*)malloc((size_t)(kmax + 1) * sizeof(int));
  int cnt = 0;
  for (int k = 1; k <= kmax; ++k)
    if (p->in[k][0] != 0.0 || p->in[k][1] != 0.0) nz[cnt++] = k;
  for (int m = 0; m < n; ++m) {
    double s = 0.0;
    for (int i = 0; i < cnt; ++i) {
      const int k = nz[i];
      const int j = (int)(((long long)k * m) % n);
      s += p->in[k][0] * p->cs[j] - p->in[k][1] * p->sn[j];
    }
    double v = p->in[0][0] + 2.0 * s;
    if (n % 2 == 0) v += (m % 2 == 0 ? 1.0 : -1.0) * p->in[half][0];
    p->out[m] = v;
  }
  free(nz);
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  free(p->cs);
  free(p->sn);
  free(p);
}
