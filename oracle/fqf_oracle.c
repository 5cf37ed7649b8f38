/*
 * fqf_oracle.c -- FP64 CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see fqf_oracle.h).  Never linked into the
 * product library.  Compiled with -ffp-contract=off and no -march so the
 * arithmetic matches the reference build (proj/CMakeLists.txt:9, -O3, no
 * FMA on baseline x86-64) operation for operation.
 */
#include "fqf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

static _Thread_local char g_err[512];

const char* oracle_last_error(void) { return g_err; }

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return 1;
}

/* ---------------------------------------------------------------- demod -- */

/* iq.cpp:17-30 -- Hamming-windowed sinc with cutoff f_c, unit DC gain. */
void oracle_lowpass_kernel(double fc, double fs, int taps, double* h) {
  int mid = taps / 2;
  double sum = 0.0;
  for (int k = 0; k < taps; ++k) {
    double x = 2.0 * kPi * (fc / fs) * (k - mid);
    double s = k == mid ? 1.0 : sin(x) / x;
    double w = 0.54 - 0.46 * cos(2.0 * kPi * k / (taps - 1));
    h[k] = s * w;
    sum += h[k];
  }
  for (int k = 0; k < taps; ++k) h[k] /= sum;
}

/* iq.cpp:34-82 -- mix with 2*exp(-i 2 pi f_c t) at absolute times, then the
 * zero-phase FIR with zero extension past the frame edges. */
int oracle_rf_to_iq(const double* rf, int T, int E, double fs, double t0, double fc, int taps,
                    double* iq) {
  if (!(fc > 0.0)) return fail("demodulation frequency must be positive");
  if (!(fs > 2.0 * fc)) return fail("sampling rate must exceed twice the demodulation frequency");
  if (!(taps >= 3 && taps % 2 == 1)) return fail("low-pass tap count must be odd and at least 3");
  if (!(T >= 1 && E >= 1)) return fail("frame has no samples");

  double* h = (double*)malloc(sizeof(double) * (size_t)taps);
  double* car = (double*)malloc(sizeof(double) * 2 * (size_t)T);
  double* mixed = (double*)malloc(sizeof(double) * 2 * (size_t)T);
  oracle_lowpass_kernel(fc, fs, taps, h);
  int mid = taps / 2;
  for (int t = 0; t < T; ++t) {
    double th = -2.0 * kPi * fc * (t0 + t / fs);
    car[2 * t] = 2.0 * cos(th);
    car[2 * t + 1] = 2.0 * sin(th);
  }
  for (int e = 0; e < E; ++e) {
    for (int t = 0; t < T; ++t) {
      double r = rf[(size_t)t * E + e];
      mixed[2 * t] = r * car[2 * t];
      mixed[2 * t + 1] = r * car[2 * t + 1];
    }
    for (int t = 0; t < T; ++t) {
      double ar = 0.0, ai = 0.0;
      int k_lo = t + mid - (T - 1);
      if (k_lo < 0) k_lo = 0;
      int k_hi = t + mid;
      if (k_hi > taps - 1) k_hi = taps - 1;
      for (int k = k_lo; k <= k_hi; ++k) {
        ar += h[k] * mixed[2 * (t + mid - k)];
        ai += h[k] * mixed[2 * (t + mid - k) + 1];
      }
      iq[2 * ((size_t)t * E + e)] = ar;
      iq[2 * ((size_t)t * E + e) + 1] = ai;
    }
  }
  free(h);
  free(car);
  free(mixed);
  return 0;
}

/* ------------------------------------------------------------ chunk plan -- */

/* das.cpp:97-119 with split_ranges (das.cpp:38-48). */
long oracle_plan_chunks(size_t n_points, int n_angles, size_t budget, size_t* ranges) {
  if (n_points == 0) return fail("reconstruction grid is empty"), -1;
  if (n_angles <= 0) return fail("need at least one transmit"), -1;
  size_t row = 16ull * (size_t)n_angles;
  if (!(budget > row)) return fail("memory budget cannot hold one voxel across %d transmits", n_angles), -1;
  if (n_points > (size_t)-1 / row) return fail("reconstruction grid is too large to size"), -1;
  size_t bytes = row * n_points;
  size_t by_total = (bytes + budget - 1) / budget;
  size_t cap = budget / row;
  size_t by_cap = (n_points + cap - 1) / cap;
  size_t k = by_total > by_cap ? by_total : by_cap;
  if (ranges) {
    size_t base = n_points / k, rem = n_points % k, at = 0;
    for (size_t i = 0; i < k; ++i) {
      size_t len = base + (i < rem ? 1 : 0);
      ranges[2 * i] = at;
      ranges[2 * i + 1] = at + len;
      at += len;
    }
  }
  return (long)k;
}

/* ------------------------------------------------------------------- DAS -- */

static inline void cmul(double ar, double ai, double br, double bi, double* cr, double* ci) {
  *cr = ar * br - ai * bi;
  *ci = ar * bi + ai * br;
}

/* Follows das_reconstruct's arithmetic (das.cpp:143-197 matrix values,
 * das.cpp:210-222 row sums in entry order, das.cpp:309-328 angle sum and the
 * 1/A scale), evaluated per voxel without materialising the CSR matrix. */
int oracle_das(const double* rf, int F, int A, int T, int E, double fs, const double* t0,
               const double* angles, const double* el, const oracle_grid* g,
               const oracle_bf* bf, double* out, uint64_t* oow) {
  if (F < 1) return fail("no frames to reconstruct");
  if (A < 1) return fail("frames carry no transmits");
  if (!(g->dims[0] >= 1 && g->dims[1] >= 1 && g->dims[2] >= 1))
    return fail("reconstruction grid dims must be positive");
  if (!(bf->c > 0.0)) return fail("sound speed must be positive");
  if (!(bf->interp_order == 0 || bf->interp_order == 1))
    return fail("interpolation order must be 0 (nearest) or 1 (linear)");
  size_t N = (size_t)g->dims[0] * g->dims[1] * g->dims[2];
  size_t nx = (size_t)g->dims[0], ny = (size_t)g->dims[1];
  double* iq = (double*)malloc(sizeof(double) * 2 * (size_t)T * E);
  double* acc = (double*)calloc(2 * N, sizeof(double));
  double omega = 2.0 * kPi * bf->fc;
  uint64_t count = 0;
  for (int f = 0; f < F; ++f) {
    memset(acc, 0, sizeof(double) * 2 * N);
    for (int a = 0; a < A; ++a) {
      const double* frame = rf + ((size_t)f * A + a) * (size_t)T * E;
      if (oracle_rf_to_iq(frame, T, E, fs, t0[a], bf->fc, bf->lowpass_taps, iq)) {
        free(iq);
        free(acc);
        return 1;
      }
      double sina = sin(angles[a]), cosa = cos(angles[a]);
      double ref = INFINITY;
      for (int e = 0; e < E; ++e) {
        double v = el[3 * e] * sina;
        if (v < ref) ref = v;
      }
      for (size_t vi = 0; vi < N; ++vi) {
        size_t i = vi % nx, j = (vi / nx) % ny, k = vi / (nx * ny);
        double px = g->origin[0] + (double)i * g->spacing[0];
        double py = g->origin[1] + (double)j * g->spacing[1];
        double pz = g->origin[2] + (double)k * g->spacing[2];
        double ttx = (px * sina + pz * cosa - ref) / bf->c;
        double sr = 0.0, si = 0.0;
        for (int e = 0; e < E; ++e) {
          double ex = el[3 * e], ey = el[3 * e + 1], ez = el[3 * e + 2];
          if (bf->f_number > 0.0) {
            double lat = hypot(px - ex, py - ey);
            if (lat * 2.0 * bf->f_number > pz - ez) continue;
          }
          double dx = px - ex, dy = py - ey, dz = pz - ez;
          double r = sqrt(dx * dx + dy * dy + dz * dz);
          double tau = ttx + r / bf->c;
          double s = (tau - t0[a]) * fs;
          double rr = cos(omega * tau), ri = sin(omega * tau);
          int live = 0;
          double pr, pi;
          if (bf->interp_order == 0) {
            double idx = round(s);
            if (idx >= 0.0 && idx < T) {
              const double* q = iq + 2 * ((size_t)idx * E + e);
              cmul(rr, ri, q[0], q[1], &pr, &pi);
              sr += pr;
              si += pi;
              live = 1;
            }
          } else {
            double sfl = floor(s);
            double frac = s - sfl;
            if (sfl >= 0.0 && sfl < T) {
              const double* q = iq + 2 * ((size_t)sfl * E + e);
              cmul((1.0 - frac) * rr, (1.0 - frac) * ri, q[0], q[1], &pr, &pi);
              sr += pr;
              si += pi;
              live = 1;
            }
            double snd = sfl + 1.0;
            if (frac > 0.0 && snd >= 0.0 && snd < T) {
              const double* q = iq + 2 * ((size_t)snd * E + e);
              cmul(frac * rr, frac * ri, q[0], q[1], &pr, &pi);
              sr += pr;
              si += pi;
              live = 1;
            }
          }
          if (!live && f == 0) count++;
        }
        acc[2 * vi] += sr;
        acc[2 * vi + 1] += si;
      }
    }
    double inv = 1.0 / A;
    for (size_t vi = 0; vi < N; ++vi) {
      out[2 * ((size_t)f * N + vi)] = acc[2 * vi] * inv;
      out[2 * ((size_t)f * N + vi) + 1] = acc[2 * vi + 1] * inv;
    }
  }
  if (oow) *oow = count;
  free(iq);
  free(acc);
  return 0;
}

/* -------------------------------------------------------- power Doppler -- */

/* render.cpp:23-42. */
void oracle_power_doppler(const double* iq, int F, size_t N, double* pd) {
  for (size_t v = 0; v < N; ++v) {
    double s = 0.0;
    for (int f = 0; f < F; ++f) {
      double re = iq[2 * ((size_t)f * N + v)], im = iq[2 * ((size_t)f * N + v) + 1];
      s += re * re + im * im;
    }
    pd[v] = s;
  }
}

/* ------------------------------------------------------------ SVD filter -- */

static int check_filter(int F, size_t N, int lo, int hi, const double* iq) {
  if (F < 1) return fail("svd_filter needs a nonempty ensemble");
  if (N == 0) return fail("svd_filter needs a nonempty grid");
  if (F < 2) return fail("svd_filter needs at least two frames");
  if ((size_t)F > N) return fail("svd_filter needs at least as many voxels as frames");
  if (!(lo >= 1 && lo <= hi && hi <= F))
    return fail("retained band must satisfy 1 <= lo <= hi <= frames, got [%d, %d] with %d frames",
                lo, hi, F);
  double nrm = 0.0;
  for (size_t i = 0; i < 2 * (size_t)F * N; ++i) nrm += iq[i] * iq[i];
  if (!(nrm > 0.0)) return fail("svd_filter needs a nonzero ensemble");
  return 0;
}

/* Descending order of w with a stable index tie-break. */
static void sort_desc(const double* w, int F, int* order) {
  for (int i = 0; i < F; ++i) order[i] = i;
  for (int i = 1; i < F; ++i) {
    int x = order[i], j = i - 1;
    while (j >= 0 && w[order[j]] < w[x]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = x;
  }
}

/* Y[f][v] = sum_j A[j][v] conj(V[f][j]) over the band columns j (A holds the
 * scaled left vectors a_j = sigma_j u_j, V the right vectors). */
static void rebuild(const double* acol, const double* V, int F, size_t N, const int* order, int lo,
                    int hi, double* out) {
  for (int f = 0; f < F; ++f)
    for (size_t v = 0; v < N; ++v) {
      double yr = 0.0, yi = 0.0;
      for (int b = lo - 1; b < hi; ++b) {
        int j = order[b];
        double ar = acol[2 * ((size_t)j * N + v)], ai = acol[2 * ((size_t)j * N + v) + 1];
        double vr = V[2 * ((size_t)f * F + j)], vi = -V[2 * ((size_t)f * F + j) + 1];
        yr += ar * vr - ai * vi;
        yi += ar * vi + ai * vr;
      }
      out[2 * ((size_t)f * N + v)] = yr;
      out[2 * ((size_t)f * N + v) + 1] = yi;
    }
}

/* svd.cpp:29-93.  Eigen's JacobiSVD is restated as a one-sided (Hestenes)
 * complex Jacobi SVD on the Casorati columns; the rebuild, the singular
 * spectrum and the |U| Pearson report follow svd.cpp:49-81. */
int oracle_svd_filter(const double* iq, int F, size_t N, int lo, int hi, double* out,
                      double* sigma, double* corr) {
  if (check_filter(F, N, lo, hi, iq)) return 1;
  size_t nel = 2 * (size_t)F * N;
  double* a = (double*)malloc(sizeof(double) * nel);
  memcpy(a, iq, sizeof(double) * nel);
  double* V = (double*)calloc(2 * (size_t)F * F, sizeof(double));
  for (int i = 0; i < F; ++i) V[2 * ((size_t)i * F + i)] = 1.0;

  for (int sweep = 0; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < F - 1; ++p)
      for (int q = p + 1; q < F; ++q) {
        double* ap = a + 2 * (size_t)p * N;
        double* aq = a + 2 * (size_t)q * N;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (size_t k = 0; k < N; ++k) {
          double pr = ap[2 * k], pi = ap[2 * k + 1], qr = aq[2 * k], qi = aq[2 * k + 1];
          al += pr * pr + pi * pi;
          be += qr * qr + qi * qi;
          gr += pr * qr + pi * qi; /* conj(ap) * aq */
          gi += pr * qi - pi * qr;
        }
        double gm = hypot(gr, gi);
        if (gm == 0.0 || gm <= 1e-15 * sqrt(al * be)) continue;
        rotated = 1;
        double zeta = (be - al) / (2.0 * gm);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        double er = gr / gm, ei = -gi / gm; /* e^{-i phi} = conj(gamma)/|gamma| */
        for (size_t k = 0; k < N; ++k) {
          double pr = ap[2 * k], pi = ap[2 * k + 1];
          double qr = aq[2 * k] * er - aq[2 * k + 1] * ei;
          double qi = aq[2 * k] * ei + aq[2 * k + 1] * er;
          ap[2 * k] = c * pr - s * qr;
          ap[2 * k + 1] = c * pi - s * qi;
          aq[2 * k] = s * pr + c * qr;
          aq[2 * k + 1] = s * pi + c * qi;
        }
        for (int r = 0; r < F; ++r) {
          double* vp = V + 2 * ((size_t)r * F + p);
          double* vq = V + 2 * ((size_t)r * F + q);
          double pr = vp[0], pi = vp[1];
          double qr = vq[0] * er - vq[1] * ei, qi = vq[0] * ei + vq[1] * er;
          vp[0] = c * pr - s * qr;
          vp[1] = c * pi - s * qi;
          vq[0] = s * pr + c * qr;
          vq[1] = s * pi + c * qi;
        }
      }
    if (!rotated) break;
  }

  double* w = (double*)malloc(sizeof(double) * F);
  int* order = (int*)malloc(sizeof(int) * F);
  for (int j = 0; j < F; ++j) {
    double s = 0.0;
    for (size_t k = 0; k < N; ++k) {
      double re = a[2 * ((size_t)j * N + k)], im = a[2 * ((size_t)j * N + k) + 1];
      s += re * re + im * im;
    }
    w[j] = sqrt(s);
  }
  sort_desc(w, F, order);
  if (sigma)
    for (int j = 0; j < F; ++j) sigma[j] = w[order[j]];

  if (corr) {
    /* Pearson correlation of |U| columns, population SD (svd.cpp:55-75). */
    double* mean = (double*)calloc(F, sizeof(double));
    double* sd = (double*)calloc(F, sizeof(double));
    double* mag = (double*)malloc(sizeof(double) * (size_t)F * N);
    for (int jj = 0; jj < F; ++jj) {
      int j = order[jj];
      double inv = w[j] > 0.0 ? 1.0 / w[j] : 0.0;
      for (size_t k = 0; k < N; ++k) {
        double re = a[2 * ((size_t)j * N + k)] * inv, im = a[2 * ((size_t)j * N + k) + 1] * inv;
        mag[(size_t)jj * N + k] = hypot(re, im);
        mean[jj] += mag[(size_t)jj * N + k];
      }
      mean[jj] /= (double)N;
      double ss = 0.0;
      for (size_t k = 0; k < N; ++k) {
        double d = mag[(size_t)jj * N + k] - mean[jj];
        ss += d * d;
      }
      sd[jj] = sqrt(ss / (double)N);
    }
    for (int i = 0; i < F; ++i) {
      corr[(size_t)i * F + i] = 1.0;
      for (int j = i + 1; j < F; ++j) {
        double denom = sd[i] * sd[j], r = 0.0;
        if (denom > 0.0) {
          double dot = 0.0;
          for (size_t k = 0; k < N; ++k)
            dot += (mag[(size_t)i * N + k] - mean[i]) * (mag[(size_t)j * N + k] - mean[j]);
          r = dot / ((double)N * denom);
        }
        corr[(size_t)i * F + j] = r;
        corr[(size_t)j * F + i] = r;
      }
    }
    free(mean);
    free(sd);
    free(mag);
  }

  if (out) rebuild(a, V, F, N, order, lo, hi, out);
  free(a);
  free(V);
  free(w);
  free(order);
  return 0;
}

/* Cyclic complex Jacobi for a Hermitian [F][F] matrix.  Each rotation is
 * J = diag(1, e^{-i phi}) R(c, s), A <- J^H A J, V <- V J. */
void oracle_heev(double* A, int F, double* w, double* Vout) {
  double* V = (double*)calloc(2 * (size_t)F * F, sizeof(double));
  for (int i = 0; i < F; ++i) V[2 * ((size_t)i * F + i)] = 1.0;
#define AR(i, j) A[2 * ((size_t)(i) * F + (j))]
#define AI(i, j) A[2 * ((size_t)(i) * F + (j)) + 1]
  double fro = 0.0;
  for (size_t i = 0; i < 2 * (size_t)F * F; ++i) fro += A[i] * A[i];
  fro = sqrt(fro);
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < F - 1; ++p)
      for (int q = p + 1; q < F; ++q) {
        double gr = AR(p, q), gi = AI(p, q);
        double gm = hypot(gr, gi);
        double app = AR(p, p), aqq = AR(q, q);
        if (gm == 0.0 || gm <= 1e-16 * sqrt(fabs(app * aqq)) || gm <= 1e-300 * fro) continue;
        rotated = 1;
        double zeta = (aqq - app) / (2.0 * gm);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        double er = gr / gm, ei = -gi / gm; /* e^{-i phi} */
        /* columns: A <- A J */
        for (int k = 0; k < F; ++k) {
          double pr = AR(k, p), pi = AI(k, p);
          double qr = AR(k, q) * er - AI(k, q) * ei, qi = AR(k, q) * ei + AI(k, q) * er;
          AR(k, p) = c * pr - s * qr;
          AI(k, p) = c * pi - s * qi;
          AR(k, q) = s * pr + c * qr;
          AI(k, q) = s * pi + c * qi;
        }
        /* rows: A <- J^H A ; J^H rows: p = c*row_p - s*e^{+i phi}*row_q */
        for (int k = 0; k < F; ++k) {
          double pr = AR(p, k), pi = AI(p, k);
          double qr = AR(q, k) * er + AI(q, k) * ei, qi = -AR(q, k) * ei + AI(q, k) * er;
          AR(p, k) = c * pr - s * qr;
          AI(p, k) = c * pi - s * qi;
          AR(q, k) = s * pr + c * qr;
          AI(q, k) = s * pi + c * qi;
        }
        AR(p, q) = AI(p, q) = AR(q, p) = AI(q, p) = 0.0;
        AI(p, p) = AI(q, q) = 0.0;
        for (int k = 0; k < F; ++k) {
          double* vp = V + 2 * ((size_t)k * F + p);
          double* vq = V + 2 * ((size_t)k * F + q);
          double pr = vp[0], pi = vp[1];
          double qr = vq[0] * er - vq[1] * ei, qi = vq[0] * ei + vq[1] * er;
          vp[0] = c * pr - s * qr;
          vp[1] = c * pi - s * qi;
          vq[0] = s * pr + c * qr;
          vq[1] = s * pi + c * qi;
        }
      }
    if (!rotated) break;
  }
  double* d = (double*)malloc(sizeof(double) * F);
  int* order = (int*)malloc(sizeof(int) * F);
  for (int i = 0; i < F; ++i) d[i] = AR(i, i);
  sort_desc(d, F, order);
  for (int j = 0; j < F; ++j) {
    w[j] = d[order[j]];
    for (int k = 0; k < F; ++k) {
      Vout[2 * ((size_t)k * F + j)] = V[2 * ((size_t)k * F + order[j])];
      Vout[2 * ((size_t)k * F + j) + 1] = V[2 * ((size_t)k * F + order[j]) + 1];
    }
  }
#undef AR
#undef AI
  free(V);
  free(d);
  free(order);
}

int oracle_gram_filter(const double* iq, int F, size_t N, int lo, int hi, double* out,
                       double* sigma) {
  if (check_filter(F, N, lo, hi, iq)) return 1;
  double* G = (double*)calloc(2 * (size_t)F * F, sizeof(double));
  for (int i = 0; i < F; ++i)
    for (int j = i; j < F; ++j) {
      const double* xi = iq + 2 * (size_t)i * N;
      const double* xj = iq + 2 * (size_t)j * N;
      double gr = 0.0, gi = 0.0;
      for (size_t v = 0; v < N; ++v) {
        gr += xi[2 * v] * xj[2 * v] + xi[2 * v + 1] * xj[2 * v + 1];
        gi += xi[2 * v] * xj[2 * v + 1] - xi[2 * v + 1] * xj[2 * v];
      }
      G[2 * ((size_t)i * F + j)] = gr;
      G[2 * ((size_t)i * F + j) + 1] = gi;
      G[2 * ((size_t)j * F + i)] = gr;
      G[2 * ((size_t)j * F + i) + 1] = -gi;
    }
  double* w = (double*)malloc(sizeof(double) * F);
  double* V = (double*)malloc(sizeof(double) * 2 * (size_t)F * F);
  oracle_heev(G, F, w, V);
  if (sigma)
    for (int j = 0; j < F; ++j) sigma[j] = sqrt(w[j] > 0.0 ? w[j] : 0.0);
  if (out) {
    /* P = V_b V_b^H ; Y[f][v] = sum_g X[g][v] P[g][f]. */
    double* P = (double*)calloc(2 * (size_t)F * F, sizeof(double));
    for (int g = 0; g < F; ++g)
      for (int f = 0; f < F; ++f) {
        double pr = 0.0, pi = 0.0;
        for (int b = lo - 1; b < hi; ++b) {
          double ar = V[2 * ((size_t)g * F + b)], ai = V[2 * ((size_t)g * F + b) + 1];
          double br = V[2 * ((size_t)f * F + b)], bi = -V[2 * ((size_t)f * F + b) + 1];
          pr += ar * br - ai * bi;
          pi += ar * bi + ai * br;
        }
        P[2 * ((size_t)g * F + f)] = pr;
        P[2 * ((size_t)g * F + f) + 1] = pi;
      }
    for (size_t v = 0; v < N; ++v)
      for (int f = 0; f < F; ++f) {
        double yr = 0.0, yi = 0.0;
        for (int g = 0; g < F; ++g) {
          double xr = iq[2 * ((size_t)g * N + v)], xi = iq[2 * ((size_t)g * N + v) + 1];
          double pr = P[2 * ((size_t)g * F + f)], pi = P[2 * ((size_t)g * F + f) + 1];
          yr += xr * pr - xi * pi;
          yi += xr * pi + xi * pr;
        }
        out[2 * ((size_t)f * N + v)] = yr;
        out[2 * ((size_t)f * N + v) + 1] = yi;
      }
    free(P);
  }
  free(G);
  free(w);
  free(V);
  return 0;
}
