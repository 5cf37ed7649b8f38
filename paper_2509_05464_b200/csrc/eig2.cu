// eig2.cu -- Hermitian eigensolve of the F x F Casorati Gram by Householder
// tridiagonalisation + implicit QL (the LAPACK zhetd2 / EISPACK tql2 route),
// all on device in FP64.  O(F^3) once, instead of per Jacobi sweep
// (eig.cu): ~40x faster at F = 200.
//
//   tridiag_kernel   one CTA: A = Q T Q^H, Q = H(0)...H(F-2), H(k) = I - tau_k v_k v_k^H
//                    (zlarfg / zhemv / zher2 steps, zhetd2 with uplo = L); the
//                    reflectors stay in A's lower triangle, T real symmetric.
//   tql2_kernel      one thread: implicit-shift QL on (d, e) (EISPACK tql2),
//                    recording every plane rotation instead of applying it.
//   zrot_kernel      F/32 CTAs: Z = product of the recorded rotations (each CTA
//                    a block of rows; rows are independent).
//   backtrans_kernel F/32 CTAs: V = Q Z (each CTA a block of columns).
//   eig_sort_kernel  eigenvalues descending, eigenvector columns permuted.
#include <cfloat>

#include "common.cuh"

namespace fqfg {

constexpr int kTriThreads = 1024;

FQFG_DEVICE double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
FQFG_DEVICE double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// Block-wide sum of a double (all threads get the result).
FQFG_DEVICE double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];  // fixed order: deterministic
  return s;
}

// A [F][F] row-major complex128 (Hermitian; overwritten: reflectors in the
// strict lower part).  d, e [F] real; tau [F] complex.
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(double2* __restrict__ A, int F,
                                                              double* __restrict__ d,
                                                              double* __restrict__ e,
                                                              double2* __restrict__ tau_out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* v = reinterpret_cast<double2*>(smem_raw);  // [F]
  double2* w = v + F;                                 // [F]
  double* red = reinterpret_cast<double*>(w + F);     // [64]
  double* sc = red + 64;                              // scalars
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;

  for (int k = 0; k + 1 < F; ++k) {
    const int m = F - k - 1;  // length of the column below the diagonal
    // zlarfg on (alpha = A[k+1][k]; x = A[k+2:][k]).
    double ss = 0.0;
    for (int r = k + 2 + tid; r < F; r += blockDim.x) {
      double2 a = A[(size_t)r * F + k];
      ss += a.x * a.x + a.y * a.y;
    }
    const double xnorm2 = block_sum(ss, red);
    if (tid == 0) {
      double2 alpha = A[(size_t)(k + 1) * F + k];
      double beta, tr, ti, scr = 0.0, sci = 0.0;
      if (xnorm2 == 0.0 && alpha.y == 0.0) {
        beta = alpha.x;
        tr = ti = 0.0;
      } else {
        beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2), alpha.x);
        tr = (beta - alpha.x) / beta;
        ti = -alpha.y / beta;
        // scale = 1 / (alpha - beta)
        double ar = alpha.x - beta, ai = alpha.y, den = ar * ar + ai * ai;
        scr = ar / den;
        sci = -ai / den;
      }
      sc[0] = beta;
      sc[1] = tr;
      sc[2] = ti;
      sc[3] = scr;
      sc[4] = sci;
      e[k] = beta;
      d[k] = A[(size_t)k * F + k].x;
      tau_out[k] = make_double2(tr, ti);
    }
    __syncthreads();
    const double2 tau = make_double2(sc[1], sc[2]);
    const double2 scale = make_double2(sc[3], sc[4]);
    // v = (1, scale * x); stored back into A's column k (reflector storage).
    for (int r = k + 1 + tid; r < F; r += blockDim.x) {
      double2 vr;
      if (r == k + 1) {
        vr = make_double2(1.0, 0.0);
      } else {
        vr = cmul(scale, A[(size_t)r * F + k]);
        A[(size_t)r * F + k] = vr;
      }
      v[r - k - 1] = vr;
    }
    __syncthreads();
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    // w' = tau * A[k+1:, k+1:] v   (warp per row, coalesced across columns)
    for (int i = warp; i < m; i += nwarp) {
      const double2* row = A + (size_t)(k + 1 + i) * F + (k + 1);
      double2 acc = make_double2(0.0, 0.0);
      for (int j = lane; j < m; j += 32) {
        double2 p = cmul(row[j], v[j]);
        acc.x += p.x;
        acc.y += p.y;
      }
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) w[i] = cmul(tau, acc);
    }
    __syncthreads();
    // alpha = -1/2 tau (w'^H v); w = w' + alpha v
    double pr = 0.0, pi = 0.0;
    for (int i = tid; i < m; i += blockDim.x) {
      double2 p = cmulc(w[i], v[i]);
      pr += p.x;
      pi += p.y;
    }
    const double sr = block_sum(pr, red);
    const double si = block_sum(pi, red);
    const double2 al = cmul(make_double2(-0.5 * tau.x, -0.5 * tau.y), make_double2(sr, si));
    for (int i = tid; i < m; i += blockDim.x) {
      double2 t = cmul(al, v[i]);
      w[i].x += t.x;
      w[i].y += t.y;
    }
    __syncthreads();
    // A[k+1:, k+1:] -= v w^H + w v^H
    for (size_t idx = tid; idx < (size_t)m * m; idx += blockDim.x) {
      int i = (int)(idx / m), j = (int)(idx % m);
      double2* a = A + (size_t)(k + 1 + i) * F + (k + 1 + j);
      double2 p = cmulc(w[j], v[i]);  // v_i conj(w_j)
      double2 q = cmulc(v[j], w[i]);  // w_i conj(v_j)
      a->x -= p.x + q.x;
      a->y -= p.y + q.y;
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[F - 1] = A[(size_t)(F - 1) * F + (F - 1)].x;
    e[F - 1] = 0.0;
    tau_out[F - 1] = make_double2(0.0, 0.0);
  }
}

// EISPACK tql2 on (d, e) (e[i] couples i and i+1), recording rotations.
// rot: (c, s) per rotation; seq[q] = {l, m, first rotation index} per sweep
// (rotations run i = m-1 .. l).  status[0] = sweeps, status[1] = 0 ok / 1 fail.
__global__ void tql2_kernel(double* __restrict__ dg, double* __restrict__ eg, int F,
                            double2* __restrict__ rot, int3* __restrict__ seq, int max_rot,
                            int max_seq, int* __restrict__ status) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* d = reinterpret_cast<double*>(smem_raw);
  double* e = d + F;
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    d[i] = dg[i];
    e[i] = eg[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nseq = 0, nrot = 0, fail = 0;
    double f = 0.0, tst1 = 0.0;
    for (int l = 0; l < F && !fail; ++l) {
      int iter = 0;
      tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
      int m = l;
      while (m < F - 1) {
        if (tst1 + fabs(e[m]) == tst1) break;
        ++m;
      }
      if (m > l) {
        do {
          if (++iter > 60 || nseq >= max_seq || nrot + (m - l) > max_rot) {
            fail = 1;
            break;
          }
          double g = d[l];
          double p = (d[l + 1] - g) / (2.0 * e[l]);
          double r = sqrt(p * p + 1.0);
          if (p < 0) r = -r;
          d[l] = e[l] / (p + r);
          d[l + 1] = e[l] * (p + r);
          double dl1 = d[l + 1];
          double h = g - d[l];
          for (int i = l + 2; i < F; ++i) d[i] -= h;
          f += h;
          p = d[m];
          double c = 1.0, c2 = c, c3 = c, el1 = e[l + 1], s = 0.0, s2 = 0.0;
          seq[nseq++] = make_int3(l, m, nrot);
          for (int i = m - 1; i >= l; --i) {
            c3 = c2;
            c2 = c;
            s2 = s;
            const double ei = e[i], di = d[i];
            g = c * ei;
            h = c * p;
            // Gram entries are far from the overflow range, so the plain
            // sqrt replaces hypot here (EISPACK uses pythag/hypot).
            r = sqrt(p * p + ei * ei);
            const double ir = 1.0 / r;
            e[i + 1] = s * r;
            s = ei * ir;
            c = p * ir;
            p = c * di - s * g;
            d[i + 1] = h + s * (c * g + s * di);
            rot[nrot++] = make_double2(c, s);
          }
          p = -s * s2 * c3 * el1 * e[l] / dl1;
          e[l] = s * p;
          d[l] = c * p;
        } while (tst1 + fabs(e[l]) > tst1);
      }
      d[l] += f;
      e[l] = 0.0;
    }
    status[0] = nseq;
    status[1] = fail;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < F; i += blockDim.x) dg[i] = d[i];
}

// Z = I, then every recorded rotation in order: columns (i, i+1) of each row.
// One thread per row, rows of a CTA staged in shared memory [32][F+1].
__global__ void __launch_bounds__(32) zrot_kernel(int F, const double2* __restrict__ rot,
                                                  const int3* __restrict__ seq,
                                                  const int* __restrict__ status,
                                                  double* __restrict__ Z) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* z = reinterpret_cast<double*>(smem_raw);
  const int pitch = F + 1;  // odd row pitch: each lane on its own bank
  const int row = blockIdx.x * 32 + threadIdx.x;
  double* zr = z + threadIdx.x * pitch;
  for (int j = 0; j < F; ++j) zr[j] = (row == j) ? 1.0 : 0.0;
  const int nseq = status[0];
  for (int q = 0; q < nseq; ++q) {
    const int3 sq = seq[q];
    int at = sq.z;
    for (int i = sq.y - 1; i >= sq.x; --i, ++at) {
      const double2 cs = rot[at];
      double h = zr[i + 1];
      zr[i + 1] = cs.y * zr[i] + cs.x * h;
      zr[i] = cs.x * zr[i] - cs.y * h;
    }
  }
  if (row < F)
    for (int j = 0; j < F; ++j) Z[(size_t)row * F + j] = zr[j];
}

// V = H(0) H(1) ... H(F-2) Z, reflectors from A's lower part.  One thread
// per column, columns of a CTA staged in shared memory [F][32].
__global__ void __launch_bounds__(32) backtrans_kernel(const double2* __restrict__ A, int F,
                                                       const double2* __restrict__ tau,
                                                       const double* __restrict__ Z,
                                                       double2* __restrict__ V) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* col = reinterpret_cast<double2*>(smem_raw);  // [F][33]
  const int j = blockIdx.x * 32 + threadIdx.x;
  const bool live = j < F;
  for (int r = 0; r < F; ++r)
    col[r * 33 + threadIdx.x] = make_double2(live ? Z[(size_t)r * F + j] : 0.0, 0.0);
  for (int k = F - 2; k >= 0; --k) {
    const double2 t = tau[k];
    if (t.x == 0.0 && t.y == 0.0) continue;
    // dot = v^H col (v[k+1] = 1, v[r] = A[r][k] for r > k+1)
    double2 dot = col[(k + 1) * 33 + threadIdx.x];
    for (int r = k + 2; r < F; ++r) {
      double2 p = cmulc(A[(size_t)r * F + k], col[r * 33 + threadIdx.x]);
      dot.x += p.x;
      dot.y += p.y;
    }
    const double2 td = cmul(t, dot);
    col[(k + 1) * 33 + threadIdx.x].x -= td.x;
    col[(k + 1) * 33 + threadIdx.x].y -= td.y;
    for (int r = k + 2; r < F; ++r) {
      double2 p = cmul(A[(size_t)r * F + k], td);
      col[r * 33 + threadIdx.x].x -= p.x;
      col[r * 33 + threadIdx.x].y -= p.y;
    }
  }
  if (live)
    for (int r = 0; r < F; ++r) V[(size_t)r * F + j] = col[r * 33 + threadIdx.x];
}

// Eigenvalues descending (stable), eigenvector columns permuted to match.
__global__ void eig_sort_kernel(const double* __restrict__ d, const double2* __restrict__ Vin,
                                int F, double* __restrict__ w, double2* __restrict__ Vout) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
    double wi = d[i];
    int rank = 0;
    for (int j = 0; j < F; ++j) rank += (d[j] > wi) || (d[j] == wi && j < i);
    w[rank] = wi;
    for (int r = 0; r < F; ++r) Vout[(size_t)r * F + rank] = Vin[(size_t)r * F + i];
  }
}


// ---- partial eigensolve: all eigenvalues, a few eigenvectors --------------
// For the clutter filter's rank form (project.cu: r = min(band, complement)
// <= 8 vectors) the full QL + rotation product is replaced by
//   bisect_kernel    one thread per eigenvalue: Sturm-count bisection on the
//                    real tridiagonal (d, e) to full precision (LAPACK dlaebz);
//                    eigenvalues written descending;
//   invit_kernel     one thread per requested mode: inverse iteration with the
//                    tridiagonal LU of T - lambda I with partial pivoting
//                    (dgttrf / dgttrs), 3 solves, then modified Gram-Schmidt
//                    across the requested vectors;
//   backtrans_sel_kernel  V[:, mode] = Q z for those vectors only.
// Accuracy is that of the full route (backward-stable eigenvalues, vectors
// conditioned by the eigenvalue gap).

// Number of eigenvalues of T (diag d, off-diag e2 = e^2) below x.
FQFG_DEVICE int sturm_count(const double* d, const double* e2, int F, double x, double pivmin) {
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += q < 0.0;
  for (int i = 1; i < F; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

// grid: ceil(F / 128) x 128.  d, e from tridiag_kernel (e[i] couples i, i+1).
__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int F,
                              double* __restrict__ w_desc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* d = reinterpret_cast<double*>(smem_raw);
  double* e2 = d + F;
  __shared__ double bounds[3];
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    d[i] = dg[i];
    e2[i] = i + 1 < F ? eg[i] * eg[i] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double gl = d[0], gu = d[0], emax = 0.0;
    for (int i = 0; i < F; ++i) {
      const double r = (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < F ? fabs(eg[i]) : 0.0);
      gl = fmin(gl, d[i] - r);
      gu = fmax(gu, d[i] + r);
      emax = fmax(emax, i + 1 < F ? e2[i] : 0.0);
    }
    const double tnorm = fmax(fabs(gl), fabs(gu));
    bounds[0] = gl - 2.0 * DBL_EPSILON * tnorm - 1e-300;
    bounds[1] = gu + 2.0 * DBL_EPSILON * tnorm + 1e-300;
    bounds[2] = fmax(DBL_MIN, DBL_MIN * emax);  // pivmin (dstebz)
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // k-th smallest
  if (k >= F) return;
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  for (int it = 0; it < 2100; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(d, e2, F, mid, pivmin) > k) hi = mid;
    else lo = mid;
  }
  w_desc[F - 1 - k] = 0.5 * (lo + hi);
}

constexpr int kInvitMax = 8;
constexpr int kInvitMaxF = 1024;

// One thread per requested mode (modes[t]: index into the descending
// eigenvalues); z [F][r] real output.  scr: 6 F r doubles of scratch (the
// LU factors and iterate of each thread live in global memory, so F is not
// bounded by a per-thread stack: F = 400 at config D).
__global__ void __launch_bounds__(32) invit_kernel(const double* __restrict__ dg,
                                                   const double* __restrict__ eg, int F,
                                                   const double* __restrict__ w_desc,
                                                   const int* __restrict__ modes, int r,
                                                   double* __restrict__ z,
                                                   double* __restrict__ scr) {
  const int t = threadIdx.x;
  if (t < r) {
    double* b = scr + (size_t)t * 6 * F;
    double* c = b + F;
    double* du2 = c + F;
    double* l = du2 + F;
    double* x = l + F;
    double* swd = x + F;  // pivot flags (0 / 1)
    const double lam = w_desc[modes[t]];
    double tnorm = 0.0;
    for (int i = 0; i < F; ++i)
      tnorm = fmax(tnorm, fabs(dg[i]) + (i > 0 ? fabs(eg[i - 1]) : 0.0) +
                              (i + 1 < F ? fabs(eg[i]) : 0.0));
    const double tiny = fmax(DBL_EPSILON * tnorm, DBL_MIN);
    // LU of T - lam I with partial pivoting: diagonals b, c (upper), du2,
    // multipliers l, pivot flags (dgttrf).
    for (int i = 0; i < F; ++i) {
      b[i] = dg[i] - lam;
      c[i] = i + 1 < F ? eg[i] : 0.0;
      du2[i] = 0.0;
      swd[i] = 0.0;
    }
    for (int i = 0; i + 1 < F; ++i) {
      const double a = eg[i];  // sub-diagonal of row i + 1
      if (fabs(b[i]) >= fabs(a)) {
        swd[i] = 0.0;
        if (b[i] == 0.0) b[i] = tiny;
        l[i] = a / b[i];
        b[i + 1] -= l[i] * c[i];
      } else {
        swd[i] = 1.0;
        l[i] = b[i] / a;
        b[i] = a;
        const double tmp = b[i + 1];
        b[i + 1] = c[i] - l[i] * tmp;
        if (i + 2 < F) {
          du2[i] = c[i + 1];
          c[i + 1] = -l[i] * du2[i];
        }
        c[i] = tmp;
      }
    }
    if (b[F - 1] == 0.0) b[F - 1] = tiny;
    for (int i = 0; i < F; ++i)
      if (fabs(b[i]) < tiny) b[i] = copysign(tiny, b[i]);
    // start vector: not orthogonal to any eigenvector in practice
    for (int i = 0; i < F; ++i) x[i] = 1.0 + 0.03125 * (double)((i * 7919 + t * 104729) % 17);
    for (int it = 0; it < 3; ++it) {
      // L solve (dgttrs, no transpose)
      for (int i = 0; i + 1 < F; ++i) {
        if (swd[i] == 0.0) {
          x[i + 1] -= l[i] * x[i];
        } else {
          const double tmp = x[i];
          x[i] = x[i + 1];
          x[i + 1] = tmp - l[i] * x[i];
        }
      }
      // U solve
      x[F - 1] /= b[F - 1];
      if (F > 1) x[F - 2] = (x[F - 2] - c[F - 2] * x[F - 1]) / b[F - 2];
      for (int i = F - 3; i >= 0; --i) x[i] = (x[i] - c[i] * x[i + 1] - du2[i] * x[i + 2]) / b[i];
      double nrm = 0.0;
      for (int i = 0; i < F; ++i) nrm = fmax(nrm, fabs(x[i]));
      const double s = nrm > 0.0 ? 1.0 / nrm : 1.0;
      for (int i = 0; i < F; ++i) x[i] *= s;
    }
    double n2 = 0.0;
    for (int i = 0; i < F; ++i) n2 += x[i] * x[i];
    const double s = 1.0 / sqrt(n2);
    for (int i = 0; i < F; ++i) x[i] *= s;
  }
  __syncwarp();
  if (t == 0) {  // modified Gram-Schmidt across the requested vectors (clusters)
    for (int a = 0; a < r; ++a) {
      double* za = scr + (size_t)a * 6 * F + 4 * F;
      for (int q = 0; q < a; ++q) {
        const double* zq = scr + (size_t)q * 6 * F + 4 * F;
        double dot = 0.0;
        for (int i = 0; i < F; ++i) dot += zq[i] * za[i];
        for (int i = 0; i < F; ++i) za[i] -= dot * zq[i];
      }
      double n2 = 0.0;
      for (int i = 0; i < F; ++i) n2 += za[i] * za[i];
      const double s = 1.0 / sqrt(n2);
      for (int i = 0; i < F; ++i) za[i] *= s;
    }
  }
  __syncwarp();
  if (t < r) {
    const double* x = scr + (size_t)t * 6 * F + 4 * F;
    for (int i = 0; i < F; ++i) z[(size_t)i * r + t] = x[i];
  }
}

// V[:, modes[t]] = H(0) ... H(F-2) z_t: one warp per requested vector, the
// reflector dot products and updates spread over the lanes (rows).
__global__ void backtrans_sel_kernel(const double2* __restrict__ A, int F,
                                     const double2* __restrict__ tau,
                                     const double* __restrict__ z, int r,
                                     const int* __restrict__ modes, double2* __restrict__ V) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (t >= r) return;
  double2* col = reinterpret_cast<double2*>(smem_raw) + (size_t)t * F;
  for (int row = lane; row < F; row += 32) col[row] = make_double2(z[(size_t)row * r + t], 0.0);
  __syncwarp();
  for (int k = F - 2; k >= 0; --k) {
    const double2 tk = tau[k];
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    // dot = v^H col, v[k+1] = 1, v[row] = A[row][k] for row > k + 1
    double2 dot = make_double2(0.0, 0.0);
    for (int row = k + 1 + lane; row < F; row += 32) {
      const double2 c = col[row];
      const double2 p = row == k + 1 ? c : cmulc(A[(size_t)row * F + k], c);
      dot.x += p.x;
      dot.y += p.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
      dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
      dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
    }
    const double2 td = cmul(tk, dot);
    for (int row = k + 1 + lane; row < F; row += 32) {
      const double2 p = row == k + 1 ? td : cmul(A[(size_t)row * F + k], td);
      col[row].x -= p.x;
      col[row].y -= p.y;
    }
    __syncwarp();
  }
  const int m = modes[t];
  for (int row = lane; row < F; row += 32) V[(size_t)row * F + m] = col[row];
}

}  // namespace fqfg
