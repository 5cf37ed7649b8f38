// demod.cu -- RF -> complex baseband (rf_to_iq, proj/src/beamform/iq.cpp:34-82),
// written straight into the frames-innermost layout the DAS kernel gathers
// from.
//
// demod_fused_kernel (the default, FIR up to kFusedMaxTaps taps) does both
// in one pass without a staging buffer; the two-kernel form below serves
// longer filters.
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
#include <cuda_fp16.h>

#include "common.cuh"

namespace fqfg {

// Where the RF of a demodulation launch lives: frame f (pass-relative, f >=
// f_base) of angle a, sample t at rf + (f - f_base) fst + a sst + (t - t0) E.
// Samples outside [t0, t0 + rows) are not stored and read as zero -- only the
// window fqfg_das_slab_samples names is uploaded, and it covers the FIR
// support of every IQ row the launch writes.  A resident [F][A][T][E]
// ensemble is fst = A T E, sst = T E, t0 = 0, rows = T.
struct RfSrc {
  const float* rf;
  long long fst, sst;
  int t0, rows;
  int f_base;  // first pass frame of the launch (a multiple of 16 for the fused kernel)
};

constexpr int kDemodTB = 64;  // output samples per CTA (8 warps x 8)

// grid: (ceil(T / 64), ceil(E / 32), F * A); block 256.
// smem: float2 mixed[(64 + taps - 1)][32], float h[taps].
// t_block0: first output block (a depth slab only needs its delay window).
// grid.z: frames [src.f_base, src.f_base + gridDim.z / A) of the pass x A;
// out is the pass's staging [fpass][A][T][E].
__global__ void __launch_bounds__(256) demod_fir_kernel(const RfSrc src,
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

  const int a = blockIdx.z % A;
  const int fl = blockIdx.z / A;                       // frame within the launch
  const int fa = (src.f_base + fl) * A + a;            // staging slice
  const int t_lo = (blockIdx.x + t_block0) * kDemodTB;
  const int e0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* sl = src.rf + (long long)fl * src.fst + (long long)a * src.sst;
  const int tlo = max(src.t0, 0), thi = min(src.t0 + src.rows, T);
  const double2* car = carrier + (size_t)a * T;

  for (int k = threadIdx.x; k < taps; k += blockDim.x) h[k] = h_g[k];
  // Input samples t' = t_lo - mid + r, r in [0, rows); zero outside [0, T)
  // (the zero extension of iq.cpp:74-76).
  for (int r = warp; r < rows; r += 8) {
    int t = t_lo - mid + r;
    int e = e0 + lane;
    float2 m = make_float2(0.f, 0.f);
    if (t >= tlo && t < thi && e < E) {
      double v = (double)__ldg(sl + (long long)(t - src.t0) * E + e);
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
__global__ void __launch_bounds__(256) demod_pack_kernel(const float2* __restrict__ stage,
                                                         float2* __restrict__ dst, int T, int E,
                                                         int A, int nf, int fpass, int row0,
                                                         int iq_row0, int iq_rows) {
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
    float2* o = dst + (((size_t)a * E + e) * (size_t)iq_rows + (row - iq_row0)) * fpass;
    for (int fl = lane; fl < fpass; fl += 32) o[fl] = tile[fl * 33 + el];
  }
}

// Fused demodulation: mix + FIR + transpose in one pass, no staging buffer.
// grid: (frame groups of kFusedG, row blocks of kFusedRB, A * ceil(E / 32));
// block 256.  A CTA owns output rows [row_lo + 32 by, +32) (row = t + 1) of
// 32 elements of angle a and frames [16 bx, 16 bx + 16) of the pass, which
// it walks two frames at a time with the next pair's RF in flight:
//   raw[2][2][32 + taps - 1][32]  f32     RF windows, cp.async double buffer
//   mixed[2][32 + taps - 1][32]   float2  FP64 mix with the carrier
//   outT[32 e][32 rows][4 frames] float2  (e stride 129: conflict-free)
// Every 4 frames outT goes out as 32-byte segments of the DAS rows
// dst[a][e][row][f .. f + 3]; the CTA completes each 128-byte line before
// it retires (L2 merges the sectors).  Guard rows and frames >= nf are zeros.
// The FIR is the same k-order FMA chain as demod_fir_kernel (bitwise equal).
constexpr int kFusedRB = 32;
constexpr int kFusedG = 16;
constexpr int kFusedOS = 129;   // outT element stride in float2 (32 rows x 4 frames + 1)
constexpr int kFusedMaxTaps = 97;
__host__ __device__ inline size_t fused_demod_smem(int taps) {
  const size_t wrows = kFusedRB + taps - 1;
  return 4 * wrows * 32 * sizeof(float) + 2 * wrows * 32 * sizeof(float2) +
         (size_t)32 * kFusedOS * sizeof(float2) + wrows * sizeof(double2) +
         (size_t)taps * sizeof(float);
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}

// H16: the tensor-core DAS layout instead (das_tc.cu): dst16[a][e][TP / 4]
// [plane hi | lo][frame][4 rows][re, im] fp16 of x S_f (scale[frame of the
// pass]), the stored rows iq_row0 .. iq_row0 + TP - 1 (rows past row_hi zero).
template <bool K33, bool H16 = false>
__global__ void __launch_bounds__(256, 2)
    demod_fused_kernel(const RfSrc src, float2* __restrict__ dst,
                       const double2* __restrict__ carrier, const float* __restrict__ h_g, int T,
                       int E, int A, int taps, int nf, int fpass, int row_lo, int row_hi,
                       int iq_row0, int iq_rows, __half* __restrict__ dst16 = nullptr,
                       const float* __restrict__ scale = nullptr, int TP = 0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int mid = K33 ? 16 : taps / 2;
  const int wrows = K33 ? 64 : kFusedRB + taps - 1;
  float* raw = reinterpret_cast<float*>(smem_raw);                // [2][2][wrows][32]
  float2* mixed = reinterpret_cast<float2*>(raw + 4 * wrows * 32);  // [2][wrows][32]
  float2* outT = mixed + (size_t)2 * wrows * 32;                   // [32][129]
  double2* car_s = reinterpret_cast<double2*>(outT + 32 * kFusedOS);  // [wrows]
  float* h = reinterpret_cast<float*>(car_s + wrows);              // [taps]
  const int ne = (E + 31) / 32;
  const int f0 = src.f_base + blockIdx.x * kFusedG;
  const int r0 = row_lo + blockIdx.y * kFusedRB;
  const int a = blockIdx.z / ne, e0 = (blockIdx.z % ne) * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = e0 + lane;
  // Input window of output row r0 + j: t' = r0 - 1 + j + mid - k; window
  // index r = j + 2 mid - k over t' = r0 - 1 - mid + r.
  const int tw0 = r0 - 1 - mid;
  const int nfr = fpass - f0 < kFusedG ? fpass - f0 : kFusedG;
  const int npair = (nfr + 1) / 2;

  // K33: rows warp + 8 j (j < 8) of the pair's two frames; row validity is
  // fixed per CTA (bit j), frame validity per pair.
  const float* rf = src.rf;
  const long long ate = src.fst;
  const int tlo = max(src.t0, 0), thi = min(src.t0 + src.rows, T);
  const float* rbase = rf + (long long)(f0 - src.f_base) * src.fst + (long long)a * src.sst +
                       (long long)(tw0 + warp - src.t0) * E + e;
  unsigned rowok = 0;
  if (K33)
    for (int j = 0; j < 8; ++j) {
      const int t = tw0 + warp + 8 * j;
      rowok |= (t >= tlo && t < thi && e < E) ? 1u << j : 0u;
    }
  auto issue = [&](int pp) {
    float* rb = raw + (size_t)(pp & 1) * 2 * wrows * 32;
    if constexpr (K33) {
#pragma unroll
      for (int fs = 0; fs < 2; ++fs) {
        const bool fok = f0 + 2 * pp + fs < nf;
        const float* pf = rbase + (2 * pp + fs) * ate;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = fok && (rowok >> j & 1u);
          cp_async4(rb + (fs * 64 + warp + 8 * j) * 32 + lane, ok ? pf + 8 * j * E : rf, ok);
        }
      }
    } else {
      for (int q = warp; q < 2 * wrows; q += 8) {
        const int f = f0 + 2 * pp + (q >= wrows), t = tw0 + (q >= wrows ? q - wrows : q);
        const bool ok = f < nf && t >= tlo && t < thi && e < E;
        cp_async4(rb + q * 32 + lane,
                  ok ? rf + (long long)(f - src.f_base) * src.fst + (long long)a * src.sst +
                           (long long)(t - src.t0) * E + e
                     : rf,
                  ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  for (int k = threadIdx.x; k < taps; k += blockDim.x) h[k] = h_g[k];
  for (int r = threadIdx.x; r < wrows; r += blockDim.x) {
    const int t = tw0 + r;
    car_s[r] = t >= 0 && t < T ? carrier[(size_t)a * T + t] : make_double2(0.0, 0.0);
  }
  const int fi = warp >> 2, rb = (warp & 3) * 8;
#pragma unroll 1
  for (int pp = 0; pp < npair; ++pp) {
    if (pp + 1 < npair) issue(pp + 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    {
      const float* rb_ = raw + (size_t)(pp & 1) * 2 * wrows * 32;
      if constexpr (K33) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 c = car_s[warp + 8 * j];
#pragma unroll
          for (int fs = 0; fs < 2; ++fs) {
            const int q = fs * 64 + warp + 8 * j;
            const double x = (double)rb_[q * 32 + lane];
            mixed[q * 32 + lane] = make_float2((float)(x * c.x), (float)(x * c.y));
          }
        }
      } else {
#pragma unroll 4
        for (int q = warp; q < 2 * wrows; q += 8) {
          const double x = (double)rb_[q * 32 + lane];
          const double2 c = car_s[q >= wrows ? q - wrows : q];
          mixed[q * 32 + lane] = make_float2((float)(x * c.x), (float)(x * c.y));
        }
      }
    }
    __syncthreads();
    const float2* mx = mixed + (size_t)fi * wrows * 32;
    unsigned long long res[8];  // (re, im) of the 8 outputs
    if constexpr (K33) {
      // packed (re, im) FMA pairs: fma.rn.f32x2 rounds each lane like fmaf
      const unsigned long long* mx2 = reinterpret_cast<const unsigned long long*>(mx);
      unsigned long long wv[40], ac[8];
#pragma unroll
      for (int r = 0; r < 40; ++r) wv[r] = mx2[(rb + r) * 32 + lane];
#pragma unroll
      for (int i = 0; i < 8; ++i) ac[i] = 0ull;
#pragma unroll
      for (int k = 0; k < 33; ++k) {
        const unsigned long long hk = f2bc(h[k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) ac[i] = ffma2(hk, wv[i + 32 - k], ac[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) res[i] = ac[i];
    } else {
      float2 acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
      for (int k = 0; k < taps; ++k) {
        const float hk = h[k];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 m = mx[(rb + i + 2 * mid - k) * 32 + lane];
          acc[i].x = fmaf(hk, m.x, acc[i].x);
          acc[i].y = fmaf(hk, m.y, acc[i].y);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        res[i] = f2pk(__float_as_uint(acc[i].x), __float_as_uint(acc[i].y));
    }
    const int fl = 2 * pp + fi;  // frame within the group
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = r0 - 1 + rb + i;
      // guard rows (t = -1, t = T) and padding frames are zeros
      const bool live = t >= 0 && t < T && f0 + fl < nf;
      reinterpret_cast<unsigned long long*>(outT)[lane * kFusedOS + (rb + i) * 4 + (fl & 3)] =
          live ? res[i] : 0ull;
    }
    if (H16 && ((pp & 1) || pp + 1 == npair)) {
      __syncthreads();
      // 32 e x 8 row chunks x 4 frames: an item is one (element, chunk,
      // frame): 4 rows x (re, im) -> 16 B per plane; lanes = 4 frames x 8
      // elements (64 B runs)
      const int fq0 = f0 + (fl & ~3);
      const int NRB = TP >> 2;
      // (a thread's items share its frame: it & 3 is fixed by threadIdx)
      const int fq = threadIdx.x & 3, f = fq0 + fq;
      const float sc = f < fpass ? __ldg(scale + f) : 1.f;
#pragma unroll 1
      for (int it = threadIdx.x; it < 32 * 8 * 4; it += 256) {
        const int el = (it >> 2) & 31, rb = it >> 7;
        const int ee = e0 + el;
        const int sr0 = r0 + 4 * rb - iq_row0;  // multiple of 4
        if (ee >= E || f >= fpass || sr0 >= TP) continue;
        uint32_t hv[4], lv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 v = r0 + 4 * rb + i <= row_hi ? outT[el * kFusedOS + (4 * rb + i) * 4 + fq]
                                                     : make_float2(0.f, 0.f);
          const float xr = v.x * sc, xi = v.y * sc;
          const __half2 h = __floats2half2_rn(xr, xi);
          const float2 hf = __half22float2(h);
          const __half2 l = __floats2half2_rn(xr - hf.x, xi - hf.y);
          hv[i] = *reinterpret_cast<const uint32_t*>(&h);
          lv[i] = *reinterpret_cast<const uint32_t*>(&l);
        }
        const size_t o = ((((size_t)a * E + ee) * NRB + (sr0 >> 2)) * 2 * fpass + f) * 8;
        *reinterpret_cast<uint4*>(dst16 + o) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<uint4*>(dst16 + o + (size_t)fpass * 8) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
      }
    } else if ((pp & 1) || pp + 1 == npair) {
      __syncthreads();
      // 32 e x 32 rows x 4 frames; a warp writes 8 rows of one element
      // (8 x 32 B segments), lane = (row-in-8, frame).
      const int fq0 = f0 + (fl & ~3);
      const int nfo = fpass - fq0 < 4 ? fpass - fq0 : 4;
      const int s = lane >> 2, fq = lane & 3;
#pragma unroll 4
      for (int g = warp; g < 32 * 4; g += 8) {
        const int el = g >> 2, row = (g & 3) * 8 + s;
        const int ee = e0 + el, rr = r0 + row;
        if (ee < E && rr <= row_hi && fq < nfo)
          dst[(((size_t)a * E + ee) * (size_t)iq_rows + (rr - iq_row0)) * fpass + fq0 + fq] =
              outT[el * kFusedOS + row * 4 + fq];
      }
    }
  }
}

}  // namespace fqfg
