// gram.cu -- Casorati Gram G = X^H X of the clutter filter (svd.cpp:38-47
// computes the SVD of X directly; G's eigenvectors are X's right singular
// vectors, G's eigenvalues the squared singular values).
//
// X is [F][N] complex64 (frame-major = Casorati column-major).  Products of two
// f32 values are exact in FP64, so this kernel -- FP64 FMA accumulation over
// split-K voxel chunks, partials reduced in a fixed order -- gives a Gram
// that is exact to FP64 rounding and bitwise deterministic.  Square output
// tiles, upper triangle only, 4x4 complex outputs per thread.
#include "common.cuh"

namespace fqfg {

constexpr int kGK = 16;   // voxels per K step

// Output tile TB x TB (TB in {32, 40, 48, 64}, picked per F to minimise the
// padded upper-triangle work: F = 200 -> 40, 15 tiles, 1.19x the useful
// work instead of 2.04x with 64), (TB / R)^2 threads with RxR complex
// outputs each (R = 5 at TB = 40: 64 threads, two full warps); double-buffered staging of 2 x 2 x kGK x (TB + 1) double2.
// Outputs per thread per dimension: 5 for TB = 40 (64 threads, 5x5), else 4.
constexpr int gram_r(int TB) { return TB == 40 ? 5 : 4; }
constexpr size_t gram_smem(int TB) { return 2 * 2 * kGK * (TB + 1) * sizeof(double2); }
constexpr int gram_threads(int TB) { return (TB / gram_r(TB)) * (TB / gram_r(TB)); }
// resident CTAs per SM the register budget is sized for (no spills)
constexpr int gram_min_ctas(int TB) { return TB == 64 ? 2 : TB == 48 ? 2 : TB == 40 ? 4 : 6; }

// grid: (n_upper_tiles, splits); block (TB/4)^2.  Partial p of tile (bi, bj)
// -> work[split][F][F] (only that tile's entries).
template <int TB>
__global__ void __launch_bounds__(gram_threads(TB), gram_min_ctas(TB))
    gram_partial_kernel(const float2* __restrict__ x, int F, size_t N, size_t v0, size_t v1,
                        double2* __restrict__ work) {
  // Double-buffered staging: the next kGK voxels are loaded into registers
  // while the current ones are multiplied (the loads' latency was the top
  // stall of the single-buffered version), one barrier per step.
  constexpr int R = gram_r(TB), NT = gram_threads(TB), Q = TB / R;
  extern __shared__ __align__(16) unsigned char gram_smem_raw[];
  auto sa = reinterpret_cast<double2(*)[kGK][TB + 1]>(gram_smem_raw);
  auto sb = sa + 2;
  const int nb = (F + TB - 1) / TB;
  // Upper-triangle tile index -> (bi, bj), bi <= bj.
  int b = blockIdx.x, bi = 0;
  while (b >= nb - bi) {
    b -= nb - bi;
    ++bi;
  }
  const int bj = bi + b;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const size_t len = v1 - v0;
  const size_t chunk = ((len + nsplit - 1) / nsplit + kGK - 1) / kGK * kGK;
  const size_t vs = v0 + (size_t)split * chunk;
  const size_t ve = min(v1, vs + chunk);

  const int tid = threadIdx.x, tx = tid % Q, ty = tid / Q;
  double2 acc[R][R];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < R; ++c) acc[r][c] = make_double2(0.0, 0.0);

  constexpr int kPer = (TB * kGK + NT - 1) / NT;  // staged elements per thread and operand
  float2 ra[kPer], rb[kPer];
  auto fetch = [&](size_t vb) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + NT * k, f = idx / kGK, v = idx % kGK;
      const size_t vv = vb + v;
      const int fa = bi * TB + f, fb = bj * TB + f;
      const bool in = idx < TB * kGK && vv < ve;
      ra[k] = (in && fa < F) ? x[(size_t)fa * N + vv] : make_float2(0.f, 0.f);
      rb[k] = (in && fb < F) ? x[(size_t)fb * N + vv] : make_float2(0.f, 0.f);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + NT * k, f = idx / kGK, v = idx % kGK;
      if (idx < TB * kGK) {
        sa[buf][v][f] = make_double2(ra[k].x, ra[k].y);
        sb[buf][v][f] = make_double2(rb[k].x, rb[k].y);
      }
    }
  };
  if (vs < ve) {
    fetch(vs);
    stash(0);
  }
  __syncthreads();
  int cur = 0;
  for (size_t vb = vs; vb < ve; vb += kGK) {
    const bool more = vb + kGK < ve;
    if (more) fetch(vb + kGK);
#pragma unroll 4
    for (int v = 0; v < kGK; ++v) {
      double2 a[R], bb[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = sa[cur][v][ty + Q * r];
#pragma unroll
      for (int c = 0; c < R; ++c) bb[c] = sb[cur][v][tx + Q * c];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < R; ++c) {
          // conj(a) * b
          acc[r][c].x = fma(a[r].x, bb[c].x, fma(a[r].y, bb[c].y, acc[r][c].x));
          acc[r][c].y = fma(a[r].x, bb[c].y, fma(-a[r].y, bb[c].x, acc[r][c].y));
        }
    }
    if (more) stash(cur ^ 1);
    __syncthreads();
    cur ^= 1;
  }
  double2* w = work + (size_t)split * F * F;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < R; ++c) {
      int fi = bi * TB + ty + Q * r, fj = bj * TB + tx + Q * c;
      if (fi < F && fj < F) w[(size_t)fi * F + fj] = acc[r][c];
    }
}

// G[i][j] = sum over splits in order (upper blocks), mirrored Hermitian.
__global__ void gram_reduce_kernel(const double2* __restrict__ work, int F, int nsplit,
                                   double2* __restrict__ g, int accumulate, int TB) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)F * F) return;
  int i = (int)(idx / F), j = (int)(idx % F);
  int bi = i / TB, bj = j / TB;
  int si = i, sj = j;
  bool mirror = bi > bj;
  if (mirror) {
    si = j;
    sj = i;
  }
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k < nsplit; ++k) {
    double2 v = work[(size_t)k * F * F + (size_t)si * F + sj];
    s.x += v.x;
    s.y += v.y;
  }
  if (mirror) s.y = -s.y;
  if (i == j) s.y = 0.0;
  if (accumulate) {
    s.x += g[idx].x;
    s.y += g[idx].y;
  }
  g[idx] = s;
}

}  // namespace fqfg
