/* fqf_rfsim.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * FP64 C restatement of the reference's frequency-domain RF channel-data
 * simulator, proj/src/rf/simulate.cpp (simulate_rf / simulate_rf_chunked,
 * run_engine:407-503), which cannot be built here (it needs FFTW,
 * simulate.cpp:3, un-vendored and unpinned, CMakeLists.txt:16-17).
 *
 *   oracle_simulate_rf  the engine: passband (make_passband:50-67), sub-element
 *                       tiling (tile_subelements:86-102), block geometry
 *                       (precompute_block:161-196), banded recurrences with
 *                       exact re-seeding every 64 bins and the elevation factor
 *                       interpolated between exact knots 8 bins apart
 *                       (accumulate_band:218-347), block spectra summed in
 *                       block order (run_engine:452-476), Gaussian pulse
 *                       weights and the c2r inverse transform (run_engine:478-
 *                       503) -- here a direct inverse DFT, which is the same sum
 *                       FFTW evaluates (rounding differs at 1e-15).
 *   oracle_reference_rf the reference test's literal restatement
 *                       (proj/tests/test_rf.cpp:51-124): every factor from
 *                       scratch per frequency, explicit transmit sum over
 *                       sub-elements, direct inverse transform.
 *
 * Pinning: the reference test pins the engine to the literal form at 1e-12
 * (test_rf.cpp:229-261) and to within the knot-interpolation error with an
 * elevation lens (263-291); tests/test_oracle.py checks that these two
 * restatements agree the same way on the same fixtures.  Both compiled with
 * -ffp-contract=off.
 */
#include "fqf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KPI 3.14159265358979323846
#define BAND_BINS 64
#define KNOT_BINS 8
#define MIN_RANGE 1e-6
#define MIN_SINC 1e-12

static double pulse_sigma(const oracle_transducer* t) {
  return 0.5 * t->fractional_bandwidth * t->center_frequency / sqrt(2.0 * log(2.0));
}

int oracle_rf_passband(const oracle_transducer* t, double fs, double duration, int* T, int* j_lo,
                       int* j_hi, double* df) {
  if (!(fs > 0.0 && duration > 0.0)) return -1;
  *T = (int)llround(fs * duration);
  if (*T < 16) return -2;
  *df = fs / *T;
  double sigma = pulse_sigma(t);
  double span = sqrt(4.0 * log(10.0)) * sigma;
  int max_bin = (*T - 1) / 2;
  int lo = (int)ceil((t->center_frequency - span) / *df);
  int hi = (int)floor((t->center_frequency + span) / *df);
  *j_lo = lo > 1 ? lo : 1;
  *j_hi = hi < max_bin ? hi : max_bin;
  return *j_lo <= *j_hi ? 0 : -3;
}

static double elevation_factor(double ysq, double e1, double e2, double k, double core_w,
                               double tail_w) {
  double w2 = e1 + e2 / (k * k);
  double core = exp(-ysq / w2);
  return core_w * core + tail_w * sqrt(sqrt(core));
}

/* Inverse transform of the weighted, conjugated spectrum (run_engine:478-503). */
static void inverse(const double* spec, int nb, int j_lo, int T, int E, double fc, double sigma,
                    double df, double* out) {
  memset(out, 0, sizeof(double) * (size_t)T * E);
  for (int e = 0; e < E; ++e) {
    for (int j = j_lo; j < j_lo + nb; ++j) {
      double f = j * df;
      double d = (f - fc) / sigma;
      double w = exp(-0.5 * d * d) / T;
      const double* s = spec + ((size_t)(j - j_lo) * E + e) * 2;
      double in_re = s[0] * w, in_im = -s[1] * w;
      for (int m = 0; m < T; ++m) {
        long ph = ((long)j * m) % T;
        double th = 2.0 * KPI * (double)ph / T;
        out[(size_t)m * E + e] += 2.0 * (in_re * cos(th) - in_im * sin(th));
      }
    }
  }
}

int oracle_simulate_rf(const double* pos, const double* refl, size_t n_scat,
                       const oracle_transducer* t, const double* tx_delays, const double* tx_apod,
                       const oracle_medium* med, double fs, double duration,
                       size_t block_scatterers, double* out, int* n_samples, int* n_bins) {
  int T, j_lo, j_hi;
  double df;
  int rc = oracle_rf_passband(t, fs, duration, &T, &j_lo, &j_hi, &df);
  if (rc) return rc;
  const int E = t->n_elements, v = t->subelements;
  const size_t vn = (size_t)E * v;
  const int bins = j_hi - j_lo + 1;
  *n_samples = T;
  *n_bins = bins;
  if (block_scatterers == 0) block_scatterers = n_scat;

  const double c = med->c;
  const double dk = 2.0 * KPI * df / c;
  const double beta_hz = med->attenuation_db_cm_mhz * (log(10.0) / 20.0) * 1e-4;
  const double beta = beta_hz * df;
  const int elev = t->elevation_height > 0.0;
  const double wa = t->elevation_aperture_factor * t->elevation_height;
  const double inv_focus = elev ? 1.0 / t->elevation_focus : 0.0;

  double* sx = malloc(sizeof(double) * vn);
  double* sy = malloc(sizeof(double) * vn);
  double* sz = malloc(sizeof(double) * vn);
  for (int e = 0; e < E; ++e)
    for (int mu = 0; mu < v; ++mu) {
      double off = ((mu + 0.5) / v - 0.5) * 2.0 * t->half_width;
      sx[(size_t)e * v + mu] = t->xyz[3 * e] + off;
      sy[(size_t)e * v + mu] = t->xyz[3 * e + 1];
      sz[(size_t)e * v + mu] = t->xyz[3 * e + 2];
    }

  const size_t spec_len = (size_t)bins * E * 2;
  double* global = calloc(spec_len, sizeof(double));
  double* block = calloc(spec_len, sizeof(double));
  /* per pair geometry of one scatterer at a time (block order is preserved
     because bands own disjoint spectrum slices and scatterers are visited in
     cloud order within every band) */
  double *r = malloc(sizeof(double) * vn), *inv_r = malloc(sizeof(double) * vn);
  double *st_re = malloc(sizeof(double) * vn), *st_im = malloc(sizeof(double) * vn);
  double *g = malloc(sizeof(double) * vn), *inv_g = malloc(sizeof(double) * vn);
  double *ss_re = malloc(sizeof(double) * vn), *ss_im = malloc(sizeof(double) * vn);
  double *arat = malloc(sizeof(double) * vn), *el1 = malloc(sizeof(double) * vn);
  double *el2 = malloc(sizeof(double) * vn);
  double *ph_re = malloc(sizeof(double) * vn), *ph_im = malloc(sizeof(double) * vn);
  double *sp_re = malloc(sizeof(double) * vn), *sp_im = malloc(sizeof(double) * vn);
  double *att = malloc(sizeof(double) * vn), *d0 = malloc(sizeof(double) * vn);
  double *d1 = malloc(sizeof(double) * vn), *dd = malloc(sizeof(double) * vn);
  double *ctr_re = malloc(sizeof(double) * vn), *ctr_im = malloc(sizeof(double) * vn);
  double* inv_k = malloc(sizeof(double) * BAND_BINS);
  double* dph = malloc(sizeof(double) * BAND_BINS * E * 2);
  double* racc = malloc(sizeof(double) * E * 2);

  const int n_bands = (bins + BAND_BINS - 1) / BAND_BINS;
  for (size_t s0 = 0; s0 < n_scat; s0 += block_scatterers) {
    size_t s1 = s0 + block_scatterers < n_scat ? s0 + block_scatterers : n_scat;
    memset(block, 0, sizeof(double) * spec_len);
    for (int b = 0; b < n_bands; ++b) {
      const int jb0 = j_lo + b * BAND_BINS;
      const int nb = j_hi - jb0 + 1 < BAND_BINS ? j_hi - jb0 + 1 : BAND_BINS;
      const double f0 = jb0 * df;
      const double k0 = 2.0 * KPI * f0 / c;
      for (int jj = 0; jj < nb; ++jj) inv_k[jj] = c / (2.0 * KPI * (jb0 + jj) * df);
      for (int e = 0; e < E; ++e) {
        double a0 = 2.0 * KPI * f0 * tx_delays[e];
        double da = 2.0 * KPI * df * tx_delays[e];
        double cr = cos(a0), ci = sin(a0);
        double sr = cos(da), si = sin(da);
        for (int jj = 0; jj < nb; ++jj) {
          dph[((size_t)jj * E + e) * 2] = cr;
          dph[((size_t)jj * E + e) * 2 + 1] = ci;
          double nr = cr * sr - ci * si;
          ci = cr * si + ci * sr;
          cr = nr;
        }
      }
      for (size_t s = s0; s < s1; ++s) {
        const double px = pos[3 * s], py = pos[3 * s + 1], pz = pos[3 * s + 2];
        const double ysq = py * py, rs = refl[s];
        for (size_t i = 0; i < vn; ++i) {  /* precompute_block:169-193 */
          double dx = px - sx[i], dy = py - sy[i], dz = pz - sz[i];
          double rr = sqrt(dx * dx + dy * dy + dz * dz);
          rr = rr > MIN_RANGE ? rr : MIN_RANGE;
          double ir = 1.0 / rr;
          r[i] = rr;
          inv_r[i] = ir;
          double ph = dk * rr;
          st_re[i] = cos(ph);
          st_im[i] = sin(ph);
          double gg = fabs(t->half_width * dx * ir);
          gg = gg > MIN_SINC ? gg : MIN_SINC;
          g[i] = gg;
          inv_g[i] = 1.0 / gg;
          double sp = dk * gg;
          ss_re[i] = cos(sp);
          ss_im[i] = sin(sp);
          arat[i] = exp(-beta * rr);
          if (elev) {
            double a = wa * (1.0 - rr * inv_focus);
            el1[i] = a * a;
            double b2 = 2.0 * rr / wa;
            el2[i] = b2 * b2;
          }
        }
        double att_k = beta * f0 / df;
        for (size_t i = 0; i < vn; ++i) {
          double ph = k0 * r[i];
          ph_re[i] = cos(ph);
          ph_im[i] = sin(ph);
          double sp = k0 * g[i];
          sp_re[i] = cos(sp);
          sp_im[i] = sin(sp);
          att[i] = exp(-att_k * r[i]);
          if (!elev) {
            d0[i] = 1.0;
            dd[i] = 0.0;
          }
        }
        for (int sb0 = 0; sb0 < nb; sb0 += KNOT_BINS) {
          int sb1 = sb0 + KNOT_BINS < nb ? sb0 + KNOT_BINS : nb;
          if (elev) {
            int hi = sb1 < nb ? sb1 : nb - 1;
            double k_a = 2.0 * KPI * (jb0 + sb0) * df / c;
            double k_b = 2.0 * KPI * (jb0 + hi) * df / c;
            double inv_den = hi > sb0 ? 1.0 / (hi - sb0) : 0.0;
            for (size_t i = 0; i < vn; ++i) {
              double a = sb0 == 0 ? elevation_factor(ysq, el1[i], el2[i], k_a,
                                                     t->elevation_core_weight,
                                                     t->elevation_tail_weight)
                                  : d1[i];
              double bb = elevation_factor(ysq, el1[i], el2[i], k_b, t->elevation_core_weight,
                                           t->elevation_tail_weight);
              d0[i] = a;
              d1[i] = bb;
              dd[i] = (bb - a) * inv_den;
            }
          }
          for (int jj = sb0; jj < sb1; ++jj) {
            double invk = inv_k[jj];
            int dj = jj - sb0;
            for (size_t i = 0; i < vn; ++i) {
              double dir = sp_im[i] * inv_g[i] * invk;
              double amp = inv_r[i] * att[i] * (d0[i] + dd[i] * dj) * dir;
              ctr_re[i] = amp * ph_re[i];
              ctr_im[i] = amp * ph_im[i];
              double nr = ph_re[i] * st_re[i] - ph_im[i] * st_im[i];
              ph_im[i] = ph_re[i] * st_im[i] + ph_im[i] * st_re[i];
              ph_re[i] = nr;
              double ns = sp_re[i] * ss_re[i] - sp_im[i] * ss_im[i];
              sp_im[i] = sp_re[i] * ss_im[i] + sp_im[i] * ss_re[i];
              sp_re[i] = ns;
              att[i] *= arat[i];
            }
            const double* dp = dph + (size_t)jj * E * 2;
            double tx_re = 0.0, tx_im = 0.0;
            for (int e = 0; e < E; ++e) {
              double rr_ = 0.0, ri_ = 0.0;
              for (int mu = 0; mu < v; ++mu) {
                rr_ += ctr_re[(size_t)e * v + mu];
                ri_ += ctr_im[(size_t)e * v + mu];
              }
              racc[2 * e] = rr_;
              racc[2 * e + 1] = ri_;
              double w = tx_apod[e];
              tx_re += w * (dp[2 * e] * rr_ - dp[2 * e + 1] * ri_);
              tx_im += w * (dp[2 * e] * ri_ + dp[2 * e + 1] * rr_);
            }
            double cr = rs * tx_re, ci = rs * tx_im;
            double* o = block + (size_t)(jb0 - j_lo + jj) * E * 2;
            for (int e = 0; e < E; ++e) {
              o[2 * e] += cr * racc[2 * e] - ci * racc[2 * e + 1];
              o[2 * e + 1] += cr * racc[2 * e + 1] + ci * racc[2 * e];
            }
          }
        }
      }
    }
    for (size_t i = 0; i < spec_len; ++i) global[i] += block[i];
  }
  inverse(global, bins, j_lo, T, E, t->center_frequency, pulse_sigma(t), df, out);

  free(sx), free(sy), free(sz), free(global), free(block), free(r), free(inv_r), free(st_re);
  free(st_im), free(g), free(inv_g), free(ss_re), free(ss_im), free(arat), free(el1), free(el2);
  free(ph_re), free(ph_im), free(sp_re), free(sp_im), free(att), free(d0), free(d1), free(dd);
  free(ctr_re), free(ctr_im), free(inv_k), free(dph), free(racc);
  return 0;
}

/* test_rf.cpp:51-124, literally. */
int oracle_reference_rf(const double* pos, const double* refl, size_t n_scat,
                        const oracle_transducer* t, const double* tx_delays,
                        const double* tx_apod, const oracle_medium* med, double fs,
                        double duration, double* out, int* n_samples, int* n_bins) {
  int T, j_lo, j_hi;
  double df;
  int rc = oracle_rf_passband(t, fs, duration, &T, &j_lo, &j_hi, &df);
  if (rc) return rc;
  const int E = t->n_elements, v = t->subelements;
  const double fc = t->center_frequency, sigma = pulse_sigma(t);
  const double beta = med->attenuation_db_cm_mhz * (log(10.0) / 20.0) * 1e-4;
  const int bins = j_hi - j_lo + 1;
  *n_samples = T;
  *n_bins = bins;
  const size_t nsub = (size_t)E * v;
  double* sub = malloc(sizeof(double) * nsub * 3);
  for (int e = 0; e < E; ++e)
    for (int mu = 0; mu < v; ++mu) {
      sub[3 * ((size_t)e * v + mu)] = t->xyz[3 * e] + ((mu + 0.5) / v - 0.5) * 2.0 * t->half_width;
      sub[3 * ((size_t)e * v + mu) + 1] = t->xyz[3 * e + 1];
      sub[3 * ((size_t)e * v + mu) + 2] = t->xyz[3 * e + 2];
    }
  double* spec = calloc((size_t)bins * E * 2, sizeof(double));
  for (int j = j_lo; j <= j_hi; ++j) {
    double f = j * df;
    double k = 2.0 * KPI * f / med->c;
    for (size_t s = 0; s < n_scat; ++s) {
      const double* p = pos + 3 * s;
      double tx_re = 0.0, tx_im = 0.0;
      for (size_t n = 0; n < nsub; ++n) {
        /* path(p, sub[n], k, f) */
        double dx = p[0] - sub[3 * n], dy = p[1] - sub[3 * n + 1], dz = p[2] - sub[3 * n + 2];
        double r = sqrt(dx * dx + dy * dy + dz * dz);
        double x = k * t->half_width * (dx / r);
        double dir = x == 0.0 ? 1.0 : sin(x) / x;
        double delta = 1.0;
        if (t->elevation_height > 0.0) {
          double wa = t->elevation_aperture_factor * t->elevation_height;
          double near_term = wa * (1.0 - r / t->elevation_focus);
          double far_term = 2.0 * r / (k * wa);
          double w2 = near_term * near_term + far_term * far_term;
          double core = exp(-p[1] * p[1] / w2);
          delta = t->elevation_core_weight * core + t->elevation_tail_weight * pow(core, 0.25);
        }
        /* std::polar(1, k r) / r * dir * delta * exp(-beta f r), per component */
        const double at = exp(-beta * f * r);
        double pr = cos(k * r) / r * dir * delta * at, pi = sin(k * r) / r * dir * delta * at;
        double a = tx_apod[n / v];
        double th = 2.0 * KPI * f * tx_delays[n / v];
        double qr = a * cos(th), qi = a * sin(th);
        tx_re += qr * pr - qi * pi;
        tx_im += qr * pi + qi * pr;
      }
      for (int e = 0; e < E; ++e) {
        double rx_re = 0.0, rx_im = 0.0;
        for (int mu = 0; mu < v; ++mu) {
          const double* q = sub + 3 * ((size_t)e * v + mu);
          double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
          double r = sqrt(dx * dx + dy * dy + dz * dz);
          double x = k * t->half_width * (dx / r);
          double dir = x == 0.0 ? 1.0 : sin(x) / x;
          double delta = 1.0;
          if (t->elevation_height > 0.0) {
            double wa = t->elevation_aperture_factor * t->elevation_height;
            double near_term = wa * (1.0 - r / t->elevation_focus);
            double far_term = 2.0 * r / (k * wa);
            double w2 = near_term * near_term + far_term * far_term;
            double core = exp(-p[1] * p[1] / w2);
            delta = t->elevation_core_weight * core + t->elevation_tail_weight * pow(core, 0.25);
          }
          const double at = exp(-beta * f * r);
          rx_re += cos(k * r) / r * dir * delta * at;
          rx_im += sin(k * r) / r * dir * delta * at;
        }
        double cr = refl[s] * tx_re, ci = refl[s] * tx_im;
        double* o = spec + ((size_t)(j - j_lo) * E + e) * 2;
        o[0] += cr * rx_re - ci * rx_im;
        o[1] += cr * rx_im + ci * rx_re;
      }
    }
  }
  inverse(spec, bins, j_lo, T, E, fc, sigma, df, out);
  free(sub);
  free(spec);
  return 0;
}
