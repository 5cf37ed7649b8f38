// gram.cu -- Casorati Gram G = X^H X of the clutter filter (svd.cpp:38-47
// computes the SVD of X directly; G's eigenvectors are X's right singular
// vectors, G's eigenvalues the squared singular values).
//
// X is [F][N] complex64 (frame-major = Casorati column-major).  Products of two
// f32 values are exact in FP64, so this kernel -- FP64 FMA accumulation over
// split-K voxel chunks, partials reduced in a fixed order -- gives a Gram
// that is exact to FP64 rounding and bitwise deterministic.  64x64 output
// blocks, upper triangle only, 4x4 complex outputs per thread.
#include "common.cuh"

namespace fqfg {

constexpr int kGB = 64;   // output block
constexpr int kGK = 16;   // voxels per K step (2 buffers x 2 x 16 x 65 x 16 B dynamic smem)
constexpr size_t kGramSmem = 2 * 2 * kGK * (kGB + 1) * sizeof(double2);

// grid: (n_upper_blocks, splits); block 256.  Partial p of block (bi, bj) ->
// work[split][F][F] (only that block's entries).
__global__ void __launch_bounds__(256, 2) gram_partial_kernel(const float2* __restrict__ x, int F,
                                                           size_t N, size_t v0, size_t v1,
                                                           double2* __restrict__ work) {
  // Double-buffered staging: the next 16 voxels are loaded into registers
  // while the current ones are multiplied (the loads' latency was the top
  // stall of the single-buffered version), one barrier per step.
  extern __shared__ __align__(16) unsigned char gram_smem[];  // 2 x 2 x kGK x (kGB + 1) double2
  auto sa = reinterpret_cast<double2(*)[kGK][kGB + 1]>(gram_smem);
  auto sb = sa + 2;
  const int nb = (F + kGB - 1) / kGB;
  // Upper-triangle block index -> (bi, bj), bi <= bj.
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

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double2 acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = make_double2(0.0, 0.0);

  constexpr int kPer = kGB * kGK / 256;  // staged elements per thread and operand
  float2 ra[kPer], rb[kPer];
  auto fetch = [&](size_t vb) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + 256 * k, f = idx / kGK, v = idx % kGK;
      const size_t vv = vb + v;
      const int fa = bi * kGB + f, fb = bj * kGB + f;
      ra[k] = (fa < F && vv < ve) ? x[(size_t)fa * N + vv] : make_float2(0.f, 0.f);
      rb[k] = (fb < F && vv < ve) ? x[(size_t)fb * N + vv] : make_float2(0.f, 0.f);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + 256 * k, f = idx / kGK, v = idx % kGK;
      sa[buf][v][f] = make_double2(ra[k].x, ra[k].y);
      sb[buf][v][f] = make_double2(rb[k].x, rb[k].y);
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
      double2 a[4], bb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = sa[cur][v][ty + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bb[c] = sb[cur][v][tx + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
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
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int fi = bi * kGB + ty + 16 * r, fj = bj * kGB + tx + 16 * c;
      if (fi < F && fj < F) w[(size_t)fi * F + fj] = acc[r][c];
    }
}

// G[i][j] = sum over splits in order (upper blocks), mirrored Hermitian.
__global__ void gram_reduce_kernel(const double2* __restrict__ work, int F, int nsplit,
                                   double2* __restrict__ g, int accumulate) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)F * F) return;
  int i = (int)(idx / F), j = (int)(idx % F);
  int bi = i / kGB, bj = j / kGB;
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
