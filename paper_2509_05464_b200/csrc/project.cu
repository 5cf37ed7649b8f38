// project.cu -- clutter-filter projection Y = X V_b V_b^H (svd.cpp:78-81:
// U_b Sigma_b V_b^H == X V_b V_b^H) with power Doppler (render.cpp:23-42)
// fused into the epilogue: PD[v] = sum_f |Y[f][v]|^2 in FP64.
//
// Two forms, picked by the host from the band rank r_b = hi - lo + 1:
//   rank form   r = min(r_b, F - r_b) <= 8: Z = X V_r (r values per voxel,
//               FP64 accumulation of exact f32 x FP64 products), then
//               Y = Z V_r^H (band) or Y = X - Z V_r^H (complement).  The
//               default band [2, F] (config.hpp:97-98) is the rank-1
//               complement; when only PD is wanted it is ||x||^2 - |z|^2,
//               one streaming pass over X (HBM-bound), else two.
//   full form   otherwise: Y = X P with P = V_b V_b^H precomputed (F x F),
//               output frames in chunks of 16 with P staged in shared memory.
#include "common.cuh"

namespace fqfg {

constexpr int kProjMaxR = 8;

// thread per voxel; Vm [F][r] selected eigenvector columns (double2).
template <int R>
__global__ void __launch_bounds__(256) project_rank_kernel(const float2* __restrict__ x, int F,
                                                           size_t N, size_t v0, size_t v1,
                                                           const double2* __restrict__ vm,
                                                           int complement,
                                                           float2* __restrict__ y,
                                                           double* __restrict__ pd) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sv = reinterpret_cast<double2*>(smem_raw);  // [F][R]
  for (int i = threadIdx.x; i < F * R; i += blockDim.x) sv[i] = vm[i];
  __syncthreads();
  size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= v1) return;
  double2 z[R];
#pragma unroll
  for (int j = 0; j < R; ++j) z[j] = make_double2(0.0, 0.0);
  double x2 = 0.0;  // ||x||^2 of the voxel's frames
  for (int f = 0; f < F; ++f) {
    float2 xf = x[(size_t)f * N + v];
    double xr = xf.x, xi = xf.y;
    x2 = fma(xr, xr, fma(xi, xi, x2));
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double2 w = sv[f * R + j];
      z[j].x = fma(xr, w.x, fma(-xi, w.y, z[j].x));
      z[j].y = fma(xr, w.y, fma(xi, w.x, z[j].y));
    }
  }
  if (!y) {
    // PD only: with orthonormal V_r, ||X V_r V_r^H||^2 = sum_j |z_j|^2 and the
    // complement's ||X - X V_r V_r^H||^2 = ||x||^2 - sum_j |z_j|^2 -- one pass
    // over X instead of two (FP64: the cancellation costs ~1e-16 x the
    // clutter-to-signal power ratio).
    double zz = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) zz = fma(z[j].x, z[j].x, fma(z[j].y, z[j].y, zz));
    if (pd) pd[v] = complement ? fmax(x2 - zz, 0.0) : zz;
    return;
  }
  double acc = 0.0;
  for (int f = 0; f < F; ++f) {
    double yr = 0.0, yi = 0.0;
    if (complement) {
      float2 xf = x[(size_t)f * N + v];
      yr = xf.x;
      yi = xf.y;
    }
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double2 w = sv[f * R + j];  // z * conj(w)
      sr = fma(z[j].x, w.x, fma(z[j].y, w.y, sr));
      si = fma(z[j].y, w.x, fma(-z[j].x, w.y, si));
    }
    if (complement) {
      yr -= sr;
      yi -= si;
    } else {
      yr = sr;
      yi = si;
    }
    acc = fma(yr, yr, fma(yi, yi, acc));
    if (y) y[(size_t)f * N + v] = make_float2((float)yr, (float)yi);
  }
  if (pd) pd[v] = acc;
}

constexpr int kProjFC = 16;  // output frames per chunk

// Y[f][v] = sum_g X[g][v] P[g][f].  grid: ceil(len / 128); block 128.
__global__ void __launch_bounds__(128) project_full_kernel(const float2* __restrict__ x, int F,
                                                           size_t N, size_t v0, size_t v1,
                                                           const double2* __restrict__ P,
                                                           float2* __restrict__ y,
                                                           double* __restrict__ pd) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sp = reinterpret_cast<double2*>(smem_raw);  // [F][kProjFC]
  size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = v < v1;
  double acc = 0.0;
  for (int f0 = 0; f0 < F; f0 += kProjFC) {
    __syncthreads();
    for (int i = threadIdx.x; i < F * kProjFC; i += blockDim.x) {
      int g = i / kProjFC, c = i % kProjFC;
      sp[i] = (f0 + c < F) ? P[(size_t)g * F + f0 + c] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (!live) continue;
    double2 yc[kProjFC];
#pragma unroll
    for (int c = 0; c < kProjFC; ++c) yc[c] = make_double2(0.0, 0.0);
    for (int g = 0; g < F; ++g) {
      float2 xg = x[(size_t)g * N + v];
      double xr = xg.x, xi = xg.y;
#pragma unroll
      for (int c = 0; c < kProjFC; ++c) {
        double2 w = sp[g * kProjFC + c];
        yc[c].x = fma(xr, w.x, fma(-xi, w.y, yc[c].x));
        yc[c].y = fma(xr, w.y, fma(xi, w.x, yc[c].y));
      }
    }
#pragma unroll
    for (int c = 0; c < kProjFC; ++c) {
      if (f0 + c < F) {
        acc = fma(yc[c].x, yc[c].x, fma(yc[c].y, yc[c].y, acc));
        if (y) y[(size_t)(f0 + c) * N + v] = make_float2((float)yc[c].x, (float)yc[c].y);
      }
    }
  }
  if (live && pd) pd[v] = acc;
}

// Gather the r mode columns of V [F][F] into vm [F][R] (zero padded) and, for
// the full form, P = V_b V_b^H.  One block.
__global__ void select_modes_kernel(const double2* __restrict__ V, int F, const int* __restrict__ modes,
                                    int r, int R, double2* __restrict__ vm) {
  for (int i = threadIdx.x; i < F * R; i += blockDim.x) {
    int f = i / R, j = i % R;
    vm[i] = j < r ? V[(size_t)f * F + modes[j]] : make_double2(0.0, 0.0);
  }
}

__global__ void projector_kernel(const double2* __restrict__ V, int F, int lo, int hi,
                                 double2* __restrict__ P) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)F * F) return;
  int g = (int)(idx / F), f = (int)(idx % F);
  double pr = 0.0, pi = 0.0;
  for (int b = lo - 1; b < hi; ++b) {  // V[g][b] * conj(V[f][b])
    double2 a = V[(size_t)g * F + b], c = V[(size_t)f * F + b];
    pr = fma(a.x, c.x, fma(a.y, c.y, pr));
    pi = fma(a.y, c.x, fma(-a.x, c.y, pi));
  }
  P[idx] = make_double2(pr, pi);
}

// PD of an unfiltered ensemble (power_doppler, render.cpp:23-42).
__global__ void power_doppler_kernel(const float2* __restrict__ x, int F, size_t N, size_t v0,
                                     size_t v1, double* __restrict__ pd) {
  size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= v1) return;
  double acc = 0.0;
  for (int f = 0; f < F; ++f) {
    float2 xf = x[(size_t)f * N + v];
    acc += (double)xf.x * xf.x + (double)xf.y * xf.y;
  }
  pd[v] = acc;
}

// Counter-hash uniform(-1, 1) synthetic RF.
__global__ void synth_rf_kernel(float* __restrict__ rf, size_t n, unsigned long long seed) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    rf[i] = (float)((double)(z >> 40) * (2.0 / 16777216.0) - 1.0);
  }
}

}  // namespace fqfg

namespace fqfg {

// ---- SvdReport::mode_correlation on device (svd.cpp:55-75) ------------------
// |U| = |X V| / sigma per mode, column means, then the population covariance
// of the centred magnitudes, all FP64.  Deterministic: fixed-order partials.

constexpr int kMagModes = 8;

// M[j][v] = |sum_f X[f][v] V[f][j]| * inv_sigma[j]; grid (ceil(N/256), ceil(F/8)).
__global__ void __launch_bounds__(256) mode_mag_kernel(const float2* __restrict__ x, int F,
                                                       size_t N, const double2* __restrict__ V,
                                                       const double* __restrict__ inv_sigma,
                                                       double* __restrict__ M) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sv = reinterpret_cast<double2*>(smem_raw);  // [F][8]
  const int j0 = blockIdx.y * kMagModes;
  for (int i = threadIdx.x; i < F * kMagModes; i += blockDim.x) {
    int f = i / kMagModes, c = i % kMagModes;
    sv[i] = j0 + c < F ? V[(size_t)f * F + j0 + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  double2 z[kMagModes];
#pragma unroll
  for (int c = 0; c < kMagModes; ++c) z[c] = make_double2(0.0, 0.0);
  for (int f = 0; f < F; ++f) {
    float2 xf = x[(size_t)f * N + v];
    double xr = xf.x, xi = xf.y;
#pragma unroll
    for (int c = 0; c < kMagModes; ++c) {
      double2 w = sv[f * kMagModes + c];
      z[c].x = fma(xr, w.x, fma(-xi, w.y, z[c].x));
      z[c].y = fma(xr, w.y, fma(xi, w.x, z[c].y));
    }
  }
#pragma unroll
  for (int c = 0; c < kMagModes; ++c)
    if (j0 + c < F) M[(size_t)(j0 + c) * N + v] = hypot(z[c].x, z[c].y) * inv_sigma[j0 + c];
}

// Per-block column sums: part[b][j] = sum of M[j][v] over the block's voxels.
__global__ void col_sum_kernel(const double* __restrict__ M, int F, size_t N, size_t chunk,
                               double* __restrict__ part) {
  const int j = blockIdx.y;
  const size_t v0 = (size_t)blockIdx.x * chunk, v1 = min(N, v0 + chunk);
  double s = 0.0;
  for (size_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) s += M[(size_t)j * N + v];
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)blockIdx.x * F + j] = red[0];
}

// Centred cross products over a voxel chunk: part[b][i][j] (32x32 output tiles).
__global__ void __launch_bounds__(256) centred_cov_kernel(const double* __restrict__ M, int F,
                                                          size_t N, size_t chunk,
                                                          const double* __restrict__ mean,
                                                          double* __restrict__ part) {
  __shared__ double sa[16][33], sb[16][33];
  const int bi = blockIdx.y, bj = blockIdx.z;
  const size_t v0 = (size_t)blockIdx.x * chunk, v1 = min(N, v0 + chunk);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[2][2] = {{0, 0}, {0, 0}};
  for (size_t vb = v0; vb < v1; vb += 16) {
    for (int i = threadIdx.x; i < 16 * 32; i += 256) {
      int vv = i / 32, c = i % 32;
      size_t v = vb + vv;
      int fa = bi * 32 + c, fb = bj * 32 + c;
      sa[vv][c] = (v < v1 && fa < F) ? M[(size_t)fa * N + v] - mean[fa] : 0.0;
      sb[vv][c] = (v < v1 && fb < F) ? M[(size_t)fb * N + v] - mean[fb] : 0.0;
    }
    __syncthreads();
    for (int vv = 0; vv < 16; ++vv)
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[r][c] = fma(sa[vv][ty + 16 * r], sb[vv][tx + 16 * c], acc[r][c]);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      int fi = bi * 32 + ty + 16 * r, fj = bj * 32 + tx + 16 * c;
      if (fi < F && fj < F) part[((size_t)blockIdx.x * F + fi) * F + fj] = acc[r][c];
    }
}

}  // namespace fqfg
