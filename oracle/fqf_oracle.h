/*
 * fqf_oracle.h -- CPU restatement of the 3D-FQFlow reconstruction hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2509_05464_b200/csrc.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * library never links or calls it.
 *
 * Every function restates one reference function in plain C, in FP64, in the
 * reference's own loop order (citations are relative to /root/reference):
 *
 *   oracle_lowpass_kernel   proj/src/beamform/iq.cpp:17-30
 *   oracle_rf_to_iq         proj/src/beamform/iq.cpp:34-82
 *   oracle_plan_chunks      proj/src/beamform/das.cpp:38-48, 97-119
 *   oracle_das              proj/tests/test_beamform.cpp:73-118 (literal DAS),
 *                           which das_reconstruct (das.cpp:224-356) matches to
 *                           1e-12; delay/mask/tap rules das.cpp:143-197
 *   oracle_power_doppler    proj/src/post/render.cpp:23-42
 *   oracle_svd_filter       proj/src/post/svd.cpp:29-93 (Eigen JacobiSVD is
 *                           restated as a one-sided complex Jacobi SVD)
 *   oracle_gram_eig         FP64 Gram + cyclic Jacobi eigensolve: the same
 *                           Y = X V_b V_b^H, used for ensembles too large for
 *                           the one-sided SVD (bench baseline).
 *
 * Pinning: tests/test_oracle.py checks these against the golden vectors in
 * tests/golden/ (produced by the reference's own unmodified sources compiled
 * into oracle/_ref by oracle/Makefile, and by numpy LAPACK for the SVD).
 *
 * Layouts: RF [T][E] time-major (RfFrame, simulate.hpp:22-37); IQ interleaved
 * complex (re, im) doubles; volumes [F][N] with voxel index x-fastest
 * (GridSpec::point, das.hpp:28-32).
 */
#ifndef FQF_ORACLE_H
#define FQF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 0 = ok; nonzero = contract violation (message via oracle_last_error). */
const char* oracle_last_error(void);

void oracle_lowpass_kernel(double fc, double fs, int taps, double* h /*[taps]*/);

int oracle_rf_to_iq(const double* rf /*[T][E]*/, int T, int E, double fs, double t0, double fc,
                    int taps, double* iq /*[T][E][2]*/);

/* Returns n_chunks; ranges[2*i], ranges[2*i+1] = [begin, end) if ranges != NULL
 * (caller allocates 2*n_chunks).  -1 on a contract violation. */
long oracle_plan_chunks(size_t n_points, int n_angles, size_t budget_bytes, size_t* ranges);

typedef struct {
  int dims[3];
  double spacing[3];
  double origin[3];
} oracle_grid;

typedef struct {
  double c;
  double fc;
  double f_number;
  int interp_order;
  int lowpass_taps;
} oracle_bf;

/* Literal delay-and-sum: for every frame, angle, voxel and element.  rf is
 * [F][A][T][E]; angles/t0 per angle slot; elements [E][3].  iq_out
 * [F][N][2].  *out_of_window counts masked-in (voxel, element, angle) pairs
 * with no recorded tap (DasStats::out_of_window semantics, das.cpp:198). */
int oracle_das(const double* rf, int F, int A, int T, int E, double fs, const double* t0,
               const double* angles, const double* elements, const oracle_grid* grid,
               const oracle_bf* bf, double* iq_out, uint64_t* out_of_window);

/* PD[v] = sum_f |IQ_f[v]|^2 in frame order. iq [F][N][2]. */
void oracle_power_doppler(const double* iq, int F, size_t N, double* pd);

/* Casorati SVD filter.  iq [F][N][2] -> out [F][N][2] (may be NULL),
 * sigma [F] descending (may be NULL), corr [F*F] (may be NULL). */
int oracle_svd_filter(const double* iq, int F, size_t N, int keep_lo, int keep_hi, double* out,
                      double* sigma, double* corr);

/* FP64 Gram route: G = X^H X, Jacobi eigensolve, Y = X V_b V_b^H.  Same
 * outputs as oracle_svd_filter (corr not produced). */
int oracle_gram_filter(const double* iq, int F, size_t N, int keep_lo, int keep_hi, double* out,
                       double* sigma);

/* Hermitian eigensolve of a [F][F][2] matrix (row-major, interleaved complex)
 * by cyclic Jacobi.  w [F] descending, v [F][F][2] with column j the
 * eigenvector of w[j].  The input is overwritten. */
void oracle_heev(double* a, int F, double* w, double* v);

/* ---- RF channel-data synthesis (fqf_rfsim.c; rf/simulate.cpp) ---- */
typedef struct {
  int n_elements;
  const double* xyz;             /* [E][3] element centres */
  double half_width;             /* b */
  int subelements;               /* v */
  double pitch;
  double center_frequency;
  double fractional_bandwidth;
  double elevation_height;       /* <= 0: no lens */
  double elevation_focus;
  double elevation_core_weight;
  double elevation_tail_weight;
  double elevation_aperture_factor;
} oracle_transducer;

typedef struct {
  double c;
  double attenuation_db_cm_mhz;
  double min_fs_ratio;
} oracle_medium;

int oracle_rf_passband(const oracle_transducer* t, double fs, double duration, int* T, int* j_lo,
                       int* j_hi, double* df);
int oracle_simulate_rf(const double* pos, const double* refl, size_t n_scat,
                       const oracle_transducer* t, const double* tx_delays, const double* tx_apod,
                       const oracle_medium* med, double fs, double duration,
                       size_t block_scatterers, double* out /*[T][E]*/, int* n_samples,
                       int* n_bins);
int oracle_reference_rf(const double* pos, const double* refl, size_t n_scat,
                        const oracle_transducer* t, const double* tx_delays,
                        const double* tx_apod, const oracle_medium* med, double fs,
                        double duration, double* out, int* n_samples, int* n_bins);

#ifdef __cplusplus
}
#endif

#endif
