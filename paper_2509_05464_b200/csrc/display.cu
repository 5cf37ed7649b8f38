// display.cu -- display and scoring on the device:
// render_db / bmode / mip / ground_truth_pd (post/render.cpp:44-145) and
// metrics: MSE, PSNR, mean local SSIM (post/metrics.cpp:24-101).
//
// Arithmetic follows the reference's order with non-contracted FP64
// (__dmul_rn / __dadd_rn: the reference is built for x86-64 without FMA):
//   * render_db: dB re the peak |v| (max reduction, exact), clamp to [0, 1];
//   * mip: per-line max with the reference's NaN behaviour (best < v);
//   * ground_truth_pd: Gaussian splats truncated at 3 sigma; each voxel sums
//     its contributions in 64-bit fixed point (2^b, b = min(52, 62 -
//     ceil(log2(scatterers + 1))): integer atomics, so the result is
//     deterministic), converts to FP64 and divides by the peak;
//   * SSIM: the reference's joint Gaussian window (weights built on the host
//     with the reference's formula), window sums in (dk, dj, di) order per
//     position, then a fixed-order tree mean.
#include "common.cuh"

namespace fqfg {

constexpr int kDispThreads = 256;

// max |v| as the bit pattern of a non-negative double (order preserving).
__global__ void peak_abs_kernel(const double* __restrict__ v, size_t n,
                                unsigned long long* __restrict__ peak_bits) {
  double m = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double a = fabs(v[i]);
    m = m < a ? a : m;  // std::max(peak, |v|): NaN never wins
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double b = __shfl_xor_sync(0xffffffffu, m, o);
    m = m < b ? b : m;
  }
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(peak_bits, (unsigned long long)__double_as_longlong(m));
}

// |IQ| of complex<double> values (std::abs -> hypot).
__global__ void cabs_kernel(const double2* __restrict__ iq, size_t n, double* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = ref_hypot(iq[i].x, iq[i].y);
}

__global__ void render_db_kernel(const double* __restrict__ v, size_t n,
                                 const unsigned long long* __restrict__ peak_bits, double factor,
                                 double dr, double* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double peak = __longlong_as_double((long long)*peak_bits);
  const double mag = fabs(v[i]);
  if (mag <= 0.0) {
    out[i] = 0.0;
    return;
  }
  const double db = __dmul_rn(factor, log10(__ddiv_rn(mag, peak)));
  const double x = __ddiv_rn(__dadd_rn(db, dr), dr);
  out[i] = x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x);  // std::clamp
}

__global__ void mip_kernel(const double* __restrict__ v, int nx, int ny, int nz, int axis,
                           double* __restrict__ out) {
  const int ox = axis == 0 ? 1 : nx, oy = axis == 1 ? 1 : ny, oz = axis == 2 ? 1 : nz;
  const size_t n = (size_t)ox * oy * oz;
  size_t flat = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (flat >= n) return;
  const int i = (int)(flat % ox), j = (int)((flat / ox) % oy), k = (int)(flat / ((size_t)ox * oy));
  const int len = axis == 0 ? nx : axis == 1 ? ny : nz;
  double best = -INFINITY;
  for (int t = 0; t < len; ++t) {
    const int ii = axis == 0 ? t : i, jj = axis == 1 ? t : j, kk = axis == 2 ? t : k;
    const double x = v[(size_t)ii + (size_t)nx * ((size_t)jj + (size_t)ny * kk)];
    best = best < x ? x : best;  // std::max(best, x)
  }
  out[flat] = best;
}

struct SplatGrid {
  int nx, ny, nz;
  double ox, oy, oz, sx, sy, sz;
  double reach, reach2, inv_two_sigma2;
  double fx, inv_fx;  // fixed-point scale 2^b of the deterministic splat sums
};

// One thread per scatterer: its truncated Gaussian splat (render.cpp:118-139).
__global__ void splat_kernel(const double* __restrict__ xyz, size_t n, const SplatGrid g,
                             double* __restrict__ out) {
  size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double ux = __ddiv_rn(__dsub_rn(xyz[3 * s], g.ox), g.sx);
  const double uy = __ddiv_rn(__dsub_rn(xyz[3 * s + 1], g.oy), g.sy);
  const double uz = __ddiv_rn(__dsub_rn(xyz[3 * s + 2], g.oz), g.sz);
  const int i0 = max(0, (int)ceil(__dsub_rn(ux, g.reach)));
  const int i1 = min(g.nx - 1, (int)floor(__dadd_rn(ux, g.reach)));
  const int j0 = max(0, (int)ceil(__dsub_rn(uy, g.reach)));
  const int j1 = min(g.ny - 1, (int)floor(__dadd_rn(uy, g.reach)));
  const int k0 = max(0, (int)ceil(__dsub_rn(uz, g.reach)));
  const int k1 = min(g.nz - 1, (int)floor(__dadd_rn(uz, g.reach)));
  for (int k = k0; k <= k1; ++k)
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        const double dx = __dsub_rn(i, ux), dy = __dsub_rn(j, uy), dz = __dsub_rn(k, uz);
        const double d2 =
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        if (d2 > g.reach2) continue;
        // integer (fixed-point) sums are associative: the result does not
        // depend on the order in which scatterers arrive (byte-identical
        // reruns, as the reference's sequential loop)
        const double c = exp(-__dmul_rn(d2, g.inv_two_sigma2));
        atomicAdd(reinterpret_cast<unsigned long long*>(out) + (size_t)i +
                      (size_t)g.nx * ((size_t)j + (size_t)g.ny * k),
                  (unsigned long long)__double2ll_rn(__dmul_rn(c, g.fx)));
      }
}

__global__ void fixed_to_double_kernel(double* __restrict__ v, size_t n, double inv_fx) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long u = reinterpret_cast<const unsigned long long*>(v)[i];
  v[i] = __dmul_rn(__ull2double_rn(u), inv_fx);
}

__global__ void scale_kernel(double* __restrict__ v, size_t n,
                             const unsigned long long* __restrict__ peak_bits) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double peak = __longlong_as_double((long long)*peak_bits);
  if (peak > 0.0) v[i] = __ddiv_rn(v[i], peak);
}

// Sum of squared differences per block (fixed order), then a fixed-order
// second pass -> deterministic.
__global__ void sqdiff_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              size_t n, double* __restrict__ part) {
  __shared__ double sh[kDispThreads];
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double d = __dsub_rn(a[i], b[i]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

struct SsimGeom {
  int nx, ny, nz;
  int hx, hy, hz;   // window half sizes
  int wx, wy, wz;   // window sizes
  int vx, vy, vz;   // valid positions per axis
};

// Local SSIM at every fully interior window position (metrics.cpp:57-78).
__global__ void ssim_kernel(const double* __restrict__ a, const double* __restrict__ b,
                            const double* __restrict__ weight, const SsimGeom g,
                            double* __restrict__ local) {
  extern __shared__ double w_sh[];
  const int nw = g.wx * g.wy * g.wz;
  for (int t = threadIdx.x; t < nw; t += blockDim.x) w_sh[t] = weight[t];
  __syncthreads();
  const size_t nvalid = (size_t)g.vx * g.vy * g.vz;
  size_t pos = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nvalid) return;
  const int i = (int)(pos % g.vx) + g.hx;
  const int j = (int)((pos / g.vx) % g.vy) + g.hy;
  const int k = (int)(pos / ((size_t)g.vx * g.vy)) + g.hz;
  double ma = 0, mb = 0, aa = 0, bb = 0, ab = 0;
  int widx = 0;
  for (int dk = -g.hz; dk <= g.hz; ++dk)
    for (int dj = -g.hy; dj <= g.hy; ++dj) {
      const size_t row = (size_t)g.nx * ((size_t)(j + dj) + (size_t)g.ny * (k + dk));
      for (int di = -g.hx; di <= g.hx; ++di, ++widx) {
        const double w = w_sh[widx];
        const double va = a[row + i + di], vb = b[row + i + di];
        ma = __dadd_rn(ma, __dmul_rn(w, va));
        mb = __dadd_rn(mb, __dmul_rn(w, vb));
        aa = __dadd_rn(aa, __dmul_rn(__dmul_rn(w, va), va));
        bb = __dadd_rn(bb, __dmul_rn(__dmul_rn(w, vb), vb));
        ab = __dadd_rn(ab, __dmul_rn(__dmul_rn(w, va), vb));
      }
    }
  const double var_a = __dsub_rn(aa, __dmul_rn(ma, ma));
  const double var_b = __dsub_rn(bb, __dmul_rn(mb, mb));
  const double cov = __dsub_rn(ab, __dmul_rn(ma, mb));
  const double c1 = 1e-4, c2 = 9e-4;
  const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, ma), mb), c1),
                               __dadd_rn(__dmul_rn(2.0, cov), c2));
  const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(ma, ma), __dmul_rn(mb, mb)), c1),
                               __dadd_rn(__dadd_rn(var_a, var_b), c2));
  local[pos] = __ddiv_rn(num, den);
}

__global__ void sum_kernel(const double* __restrict__ v, size_t n, double* __restrict__ part) {
  __shared__ double sh[kDispThreads];
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    acc = __dadd_rn(acc, v[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

}  // namespace fqfg
