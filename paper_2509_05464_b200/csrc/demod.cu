// demod.cu -- RF -> complex baseband (rf_to_iq, proj/src/beamform/iq.cpp:34-82),
// written straight into the frames-innermost layout the DAS kernel gathers
// from.
//
// Two kernels:
//   demod_fir_kernel   mix with 2 exp(-i 2 pi f_c (t0 + t/fs)) (iq.cpp:51-54) and
//                      the zero-phase FIR h (iq.cpp:17-30, 70-78), one
//                      (frame, angle) slice at a time, elements on lanes.
//                      Output staging layout [frame][angle][t][element].
//   demod_pack_kernel  transpose (frame, element) tiles into the DAS layout
//                      [angle][pass][element][t + 1][frame-in-pass], zeroing
//                      the guard rows t = -1, t = T and the padding frames.
//
// Arithmetic: the carrier and filter taps are computed in FP64 on the host
// (same formulas as iq.cpp) and rounded to f32; the product RF * carrier is
// formed in FP64 and rounded; the 33-tap sum runs in f32 FMA.  Relative
// error vs the FP64 reference is ~1e-7 (tests/test_gpu_parity.py).
#include "common.cuh"

namespace fqfg {

constexpr int kDemodTB = 64;  // output samples per CTA (8 warps x 8)

// grid: (ceil(T / 64), ceil(E / 32), F * A); block 256.
// smem: float2 mixed[(64 + taps - 1)][32], float h[taps].
// t_block0: first output block (a depth slab only needs its delay window).
__global__ void __launch_bounds__(256) demod_fir_kernel(const float* __restrict__ rf,
                                                        float2* __restrict__ out,
                                                        const double2* __restrict__ carrier,
                                                        const float* __restrict__ h_g, int T,
                                                        int E, int A, int taps,
                                                        int t_block0 = 0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int mid = taps / 2;
  const int rows = kDemodTB + taps - 1;
  float2* mixed = reinterpret_cast<float2*>(smem_raw);
  float* h = reinterpret_cast<float*>(mixed + (size_t)rows * 32);

  const int fa = blockIdx.z;  // frame * A + angle
  const int a = fa % A;
  const int t_lo = (blockIdx.x + t_block0) * kDemodTB;
  const int e0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* src = rf + (size_t)fa * T * E;
  const double2* car = carrier + (size_t)a * T;

  for (int k = threadIdx.x; k < taps; k += blockDim.x) h[k] = h_g[k];
  // Input samples t' = t_lo - mid + r, r in [0, rows); zero outside [0, T)
  // (the zero extension of iq.cpp:74-76).
  for (int r = warp; r < rows; r += 8) {
    int t = t_lo - mid + r;
    int e = e0 + lane;
    float2 m = make_float2(0.f, 0.f);
    if (t >= 0 && t < T && e < E) {
      double v = (double)__ldg(src + (size_t)t * E + e);
      double2 c = car[t];
      m = make_float2((float)(v * c.x), (float)(v * c.y));
    }
    mixed[r * 32 + lane] = m;
  }
  __syncthreads();

  const int e = e0 + lane;
  float2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  // Output t = t_lo + warp*8 + i needs mixed[t + mid - k] = row (warp*8 + i +
  // 2*mid - k) ... expressed over the shared window index j = i - k + taps - 1.
  const int base = warp * 8;
  if (taps == 33) {
    // The reference default: the 8 outputs x 33 taps of this thread read 40
    // distinct window samples -- load them once into registers (6.6x fewer
    // shared-memory loads), same k-order FMA chain per output.
    float2 wv[40];
#pragma unroll
    for (int r = 0; r < 40; ++r) wv[r] = mixed[(base + r) * 32 + lane];
#pragma unroll
    for (int k = 0; k < 33; ++k) {
      const float hk = h[k];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 m = wv[i + 32 - k];
        acc[i].x = fmaf(hk, m.x, acc[i].x);
        acc[i].y = fmaf(hk, m.y, acc[i].y);
      }
    }
  } else {
    for (int k = 0; k < taps; ++k) {
      float hk = h[k];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 m = mixed[(base + i + 2 * mid - k) * 32 + lane];
        acc[i].x = fmaf(hk, m.x, acc[i].x);
        acc[i].y = fmaf(hk, m.y, acc[i].y);
      }
    }
  }
  if (e < E) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int t = t_lo + base + i;
      if (t < T) out[((size_t)fa * T + t) * E + e] = acc[i];
    }
  }
}

// grid: (T + 2 rows, ceil(E / 32), A); block 256.
// Reads the pass's staging [nf][A][T][E] float2 and writes the DAS layout
// dst[a][e][row][fl] (row = t + 1), zero for guard rows and frames >= nf.
// pairs = 1: the time-row-pair layout dst[a][e][row / 2][fl][row % 2] of the
// TMEM-window DAS (das2 mode 6), P = (T + 3) / 2 pairs per element.
__global__ void __launch_bounds__(256) demod_pack_kernel(const float2* __restrict__ stage,
                                                         float2* __restrict__ dst, int T, int E,
                                                         int A, int nf, int fpass,
                                                         int row0 = 0, int pairs = 0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* tile = reinterpret_cast<float2*>(smem_raw);  // [fpass][33]
  const int row = row0 + blockIdx.x;                    // 0 .. T+1
  const int e0 = blockIdx.y * 32;
  const int a = blockIdx.z;
  const int t = row - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool live_row = t >= 0 && t < T;
  for (int fl = warp; fl < fpass; fl += 8) {
    int e = e0 + lane;
    float2 v = make_float2(0.f, 0.f);
    if (live_row && fl < nf && e < E) v = stage[(((size_t)fl * A + a) * T + t) * E + e];
    tile[fl * 33 + lane] = v;
  }
  __syncthreads();
  for (int el = warp; el < 32; el += 8) {
    int e = e0 + el;
    if (e >= E) break;
    if (pairs) {
      float2* o = dst + ((((size_t)a * E + e) * (size_t)((T + 3) / 2) + (row >> 1)) * fpass) * 2 +
                  (row & 1);
      for (int fl = lane; fl < fpass; fl += 32) o[2 * fl] = tile[fl * 33 + el];
    } else {
      float2* o = dst + (((size_t)a * E + e) * (size_t)(T + 2) + row) * fpass;
      for (int fl = lane; fl < fpass; fl += 32) o[fl] = tile[fl * 33 + el];
    }
  }
}

}  // namespace fqfg
