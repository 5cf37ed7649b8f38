// gram_dmma.cu -- Casorati Gram G = X^H X on the FP64 tensor cores
// (mma.sync m8n8k4 f64, "DMMA"); opt-in FQFG_GRAM=dmma, same tiles, split-K
// partials and fixed-order reduction (gram_reduce_kernel) as the FP64 CUDA-core
// engine in gram.cu (svd.cpp:38-47: G's eigenvectors are X's right singular
// vectors).
//
// Products of two f32 values are exact in FP64, so each DMMA adds exact
// products; only the FP64 accumulation order differs from gram.cu.  Complex
// product conj(a) b as four real DMMAs per 8 x 8 block and 4 voxels:
//   Re += ar^T br + ai^T bi,   Im += ar^T bi + (-ai)^T br.
// Fragments (row.col m8n8k4): lane = 4 g + t holds A[g][t] and B[t][g], i.e.
// X[frame0 + g][voxel0 + t] for both operands, and C[g][2t .. 2t+1].
//
// Tile 40 x 40 frames (5 x 5 blocks) per CTA, 5 warps: warp w owns block row
// w (5 blocks, 20 FP64 accumulators).  X chunks of kDV voxels are staged in
// shared memory as float2 by cp.async (zero-filled outside [F) x [v0, v1)),
// double-buffered.
#include "common.cuh"

namespace fqfg {

constexpr int kDTB = 40;               // frames per tile side
constexpr int kDV = 32;                // voxels per stage
constexpr int kDVP = kDV + 4;          // row pitch (float2): conflict-free fragment loads
constexpr int kDWarps = kDTB / 8;      // one warp per 8-frame block row
constexpr int kDThreads = 32 * kDWarps;
constexpr size_t kDmmaSmem = (size_t)2 * 2 * kDTB * kDVP * sizeof(float2);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem),
               "r"(ok ? 8 : 0)
               : "memory");
}

// grid (n_upper_tiles, splits), block kDThreads.  Partial of tile (bi, bj)
// and split s -> work[s][F][F] (that tile's entries only), as gram.cu.
__global__ void __launch_bounds__(kDThreads)
    gram_dmma_kernel(const float2* __restrict__ x, int F, size_t N, size_t v0, size_t v1,
                     double2* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char dmma_smem_raw[];
  float2* sm = reinterpret_cast<float2*>(dmma_smem_raw);  // [buf][side][kDTB][kDVP]
  const int nb = (F + kDTB - 1) / kDTB;
  int b = blockIdx.x, bi = 0;
  while (b >= nb - bi) {
    b -= nb - bi;
    ++bi;
  }
  const int bj = bi + b;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const size_t len = v1 - v0;
  const size_t chunk = ((len + nsplit - 1) / nsplit + kDV - 1) / kDV * kDV;
  const size_t vs = v0 + (size_t)split * chunk;
  const size_t ve = min(v1, vs + chunk);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  auto stage = [&](int buf, size_t vb) {
    float2* s = sm + (size_t)buf * 2 * kDTB * kDVP;
    for (int q = tid; q < 2 * kDTB * kDV; q += kDThreads) {
      const int side = q / (kDTB * kDV), r = q % (kDTB * kDV), f = r / kDV, v = r % kDV;
      const int fr = (side ? bj : bi) * kDTB + f;
      const size_t vv = vb + v;
      const bool ok = fr < F && vv < ve;
      cp_async8(s + ((size_t)side * kDTB + f) * kDVP + v, ok ? x + (size_t)fr * N + vv : x, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  double re[kDWarps][2], im[kDWarps][2];
#pragma unroll
  for (int j = 0; j < kDWarps; ++j) re[j][0] = re[j][1] = im[j][0] = im[j][1] = 0.0;

  int cur = 0;
  if (vs < ve) stage(0, vs);
  for (size_t vb = vs; vb < ve; vb += kDV) {
    if (vb + kDV < ve) {
      stage(cur ^ 1, vb + kDV);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float2* sa = sm + (size_t)cur * 2 * kDTB * kDVP + (size_t)(w * 8 + g) * kDVP + t;
    const float2* sb = sm + ((size_t)cur * 2 + 1) * kDTB * kDVP + (size_t)g * kDVP + t;
#pragma unroll 2
    for (int k = 0; k < kDV; k += 4) {
      const float2 a = sa[k];
      const double ar = a.x, ai = a.y, nai = -ai;
#pragma unroll
      for (int j = 0; j < kDWarps; ++j) {
        const float2 bb = sb[(size_t)j * 8 * kDVP + k];
        const double br = bb.x, bim = bb.y;
        dmma(re[j][0], re[j][1], ar, br);
        dmma(im[j][0], im[j][1], ar, bim);
        dmma(re[j][0], re[j][1], ai, bim);
        dmma(im[j][0], im[j][1], nai, br);
      }
    }
    __syncthreads();  // the next iteration's stage() overwrites this buffer
    cur ^= 1;
  }
  double2* out = work + (size_t)split * F * F;
  const int fi = bi * kDTB + w * 8 + g;
  if (fi < F) {
#pragma unroll
    for (int j = 0; j < kDWarps; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int fj = bj * kDTB + j * 8 + 2 * t + e;
        if (fj < F) out[(size_t)fi * F + fj] = make_double2(re[j][e], im[j][e]);
      }
  }
}

}  // namespace fqfg
