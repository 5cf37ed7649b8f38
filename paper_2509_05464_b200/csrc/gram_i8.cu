// gram_i8.cu -- the Casorati Gram G = X^H X on the 5th-generation tensor
// cores, exact-product int8 digit splitting (Ozaki scheme): tcgen05.mma
// kind::i8 with int32 accumulation in TMEM and FP64 recombination.
//
// X [F][N] complex64 (column f of the Casorati matrix = frame f, svd.cpp:38-41)
// is read as Xr, Xi (real F x N each).  Then
//     Re G = Xr Xr^T + Xi Xi^T,   Im G = P - P^T  with  P = Xr Xi^T.
// Each frame row is scaled by a power of two 2^-e_f (max |x| < 2^e_f, one
// pass over X: gram_amax_kernel) and split into four signed 7-bit digits,
//     x 2^-e_f = d1/128 + d2/128^2 + d3/128^3 + d4/128^4 + r,
// d1 by truncation, d2..d4 by rounding to nearest (|d| <= 127, every step
// exact in f32), |r| <= 2^-28: the first 28 bits of every sample, unbiased
// below.  Products of digit levels s = d + d' <= 6 are kept (the 13 pairs
// whose weight 128^-s is at least 2^-42; the dropped ones bound the error
// near 1e-9 of the largest entry): per level an exact int32 GEMM on the
// tensor core, recombined in FP64 as 2^(e_i + e_j) sum_s 128^-s P_s.
// The int32 accumulators cannot overflow inside a K split of <= 16384
// voxels (4 pairs x 2 components x 127^2 x 16384 < 2^31).
//
// Kernels:
//   gram_amax_kernel      per-frame max |x| (bit pattern, atomicMax)
//   gram_i8_split_kernel  digits of a voxel batch -> Q [4 planes][F][K bytes],
//                         K = per 64-voxel group: 64 B of Xr digits, then 64 B
//                         of Xi digits (one 128-byte swizzle row; MMA K steps
//                         0, 1 are Xr, 2, 3 are Xi)
//   gram_i8_mma_kernel    CTA = (tile, K split): tile = 128 frames (A rows) x
//                         48 frames (B rows); TMA (SWIZZLE_128B, K-major) of
//                         the 4 planes of A and B per 64-voxel stage (full
//                         128-byte lines); one thread issues 24
//                         tcgen05.mma.kind::i8 per stage (per A digit plane
//                         one MMA over the consecutive B planes, N up to 192)
//                         into 10 TMEM accumulators (Re and P for levels
//                         2..6, 48 columns each, zeroed at the start); 4
//                         epilogue warps drain TMEM once per split into an
//                         FP64 partial
//   gram_i8_reduce_kernel G = fixed-order FP64 sum of the partials (exactly
//                         Hermitian: the integer sums commute), += G if asked
#include <cuda.h>

#include "common.cuh"

namespace fqfg {

constexpr int kI8Threads = 192;   // warp 0 TMA, warp 1 MMA (+ TMEM alloc), warps 2-5 epilogue
constexpr int kI8Stages = 2;
constexpr int kI8StageVox = 64;   // voxels per pipeline stage: one 128-byte row per plane
constexpr int kI8SplitVox = 16384;  // voxels per K split (int32 accumulator bound)
constexpr int kI8TileM = 128, kI8TileN = 48;
constexpr int kI8MaxLevel = 6;  // digit levels 2..6 (13 digit pairs)
constexpr int kI8MaxTiles = 192;  // F = 1024: 8 x 22 tiles
// shared-memory stage: A [4 planes][128 rows][128 B], B [4][48 rows][128 B]
constexpr int kI8ABytes = 4 * kI8TileM * 128;  // 64 KB
constexpr int kI8BBytes = 4 * kI8TileN * 128;  // 24 KB
constexpr int kI8StageBytes = kI8ABytes + kI8BBytes;
constexpr size_t kI8Smem = 1024 + (size_t)kI8Stages * kI8StageBytes + 256;

struct I8Gram {
  int F;
  int ntile;
  int m0[kI8MaxTiles], n0[kI8MaxTiles], nn[kI8MaxTiles];
  size_t nvox;     // voxels of this batch
  int nsplit;      // K splits of this batch
  const unsigned* amax;  // [F] bit patterns of max |x| per frame
};

// ---- per-frame max |x| over voxels [v0, v1) of x [F][ld] complex64.
__global__ void gram_amax_kernel(const float2* __restrict__ x, size_t ld, size_t v0, size_t v1,
                                 unsigned* __restrict__ amax) {
  const int f = blockIdx.y;
  const float2* row = x + (size_t)f * ld;
  float m = 0.f;
  const size_t step = (size_t)gridDim.x * blockDim.x;
  size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + 7 * step < v1; v += 8 * step) {
    float2 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __ldcs(row + v + k * step);
#pragma unroll
    for (int k = 0; k < 8; ++k) m = fmaxf(m, fmaxf(fabsf(a[k].x), fabsf(a[k].y)));
  }
  for (; v < v1; v += step) {
    const float2 a = row[v];
    m = fmaxf(m, fmaxf(fabsf(a.x), fabsf(a.y)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(amax + f, __float_as_uint(m));
}

// 2^-e with max |x| < 2^e: the row scale (0 rows: 1).
FQFG_DEVICE int frame_exp(unsigned bits) {
  if (bits == 0u) return 0;
  int e;
  frexpf(__uint_as_float(bits), &e);  // m in [0.5, 1): max < 2^e
  return e;
}

// Four digits of y (|y| < 1) packed with the digits of three more values:
// returns the byte of digit plane p.
FQFG_DEVICE void digits4(float y, int (&d)[4]) {
  float t = y * 128.f;
  float q = truncf(t);
  d[0] = (int)q;
  float r = t - q;
#pragma unroll
  for (int p = 1; p < 4; ++p) {
    t = r * 128.f;
    q = fminf(fmaxf(rintf(t), -127.f), 127.f);
    d[p] = (int)q;
    r = t - q;
  }
}

// ---- digits of voxels [vb, vb + nvox) -> Q.  Thread = (frame, 8 voxels):
// 16-byte loads when the row is 16-byte aligned, one 8-byte store per plane
// and component.  Q row pitch kb bytes = 128 x ceil(nvox / 64); voxels past
// nvox are zeros.
__global__ void __launch_bounds__(256) gram_i8_split_kernel(const float2* __restrict__ x,
                                                            size_t ld, size_t vb, size_t nvox,
                                                            const unsigned* __restrict__ amax,
                                                            int F, size_t kb,
                                                            unsigned* __restrict__ Q) {
  const int f = blockIdx.y;
  const size_t v = 8 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);  // first of 8 voxels
  if (v >= (nvox + 63) / 64 * 64) return;
  const int e = frame_exp(amax[f]);
  const float sc = ldexpf(1.f, -e);
  const float2* row = x + (size_t)f * ld + vb;
  float2 a[8];
  const bool aligned = ((reinterpret_cast<uintptr_t>(row + v)) & 15) == 0;
  if (aligned && v + 8 <= nvox) {
    const float4* r4 = reinterpret_cast<const float4*>(row + v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 q = __ldcs(r4 + k);
      a[2 * k] = make_float2(q.x, q.y);
      a[2 * k + 1] = make_float2(q.z, q.w);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = v + k < nvox ? row[v + k] : make_float2(0.f, 0.f);
  }
  unsigned long long wr[4] = {0ull, 0ull, 0ull, 0ull}, wi[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int dr[4], di[4];
    digits4(a[k].x * sc, dr);
    digits4(a[k].y * sc, di);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      wr[p] |= (unsigned long long)((unsigned)dr[p] & 0xffu) << (8 * k);
      wi[p] |= (unsigned long long)((unsigned)di[p] & 0xffu) << (8 * k);
    }
  }
  // group g = v / 64: bytes [128 g, 128 g + 64) Xr digits, [128 g + 64, 128 g + 128) Xi
  const size_t g = v / 64, off = v % 64;
  const size_t plane = (size_t)F * kb;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    unsigned char* base = reinterpret_cast<unsigned char*>(Q) + p * plane + (size_t)f * kb + 128 * g;
    *reinterpret_cast<unsigned long long*>(base + off) = wr[p];
    *reinterpret_cast<unsigned long long*>(base + 64 + off) = wi[p];
  }
}

FQFG_DEVICE uint64_t i8_desc_sw128(uint32_t saddr) {
  // K-major SWIZZLE_128B: rows of 128 B, 8-row atoms of 1024 B (SBO), version
  // 1, layout type 2; a K step of 32 B inside the atom advances the start.
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

FQFG_DEVICE void i8_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

FQFG_DEVICE void i8_commit(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a)
               : "memory");
}

FQFG_DEVICE void i8_mbar_init(uint64_t* bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

FQFG_DEVICE void i8_mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAITI8_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITI8_%=;\n}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

// 3-D TMA (bytes, frame row, digit plane) into shared memory.
FQFG_DEVICE void i8_tma3(void* dst, const CUtensorMap* map, int k, int row, int plane,
                         uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
      "l"(map), "r"(k), "r"(row), "r"(plane), "r"(b)
      : "memory");
}

// mapA: box {128 B, 128 rows, 4 planes}; mapB: box {128 B, 64 rows, 4 planes}
// (the same tensor Q [4][F][kb]; rows >= F are zero-filled by the TMA).
__global__ void __launch_bounds__(kI8Threads, 1)
    gram_i8_mma_kernel(const __grid_constant__ CUtensorMap mapA,
                       const __grid_constant__ CUtensorMap mapB, const I8Gram g,
                       double2* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kI8Stages * kI8StageBytes);
  uint64_t* empty = full + kI8Stages;
  uint64_t* accfull = empty + kI8Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x % g.ntile, split = blockIdx.x / g.ntile;
  const int m0 = g.m0[tile], n0 = g.n0[tile], nn = g.nn[tile];
  const size_t vs = (size_t)split * kI8SplitVox;
  const size_t ve = min(g.nvox, vs + kI8SplitVox);
  const int nstage = ve > vs ? (int)((ve - vs + kI8StageVox - 1) / kI8StageVox) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      i8_mbar_init(&full[s], 1);
      i8_mbar_init(&empty[s], 1);
    }
    i8_mbar_init(accfull, 1);
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 1) {
    unsigned a = (unsigned)__cvta_generic_to_shared(tmem_slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // The stacked MMAs below accumulate into level ranges that start at
  // different levels, so no single MMA can initialise them: the epilogue
  // warps zero all 512 columns of their lane quadrant first.
  if (warp >= 2) {
    const uint32_t z[32] = {0u};
    const uint32_t row = (uint32_t)(32 * (warp & 3)) << 16;
#pragma unroll 1
    for (int c = 0; c < 512; c += 32)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
              tmem + row + (uint32_t)c),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]),
          "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]),
          "r"(z[15]), "r"(z[16]), "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]),
          "r"(z[22]), "r"(z[23]), "r"(z[24]), "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]),
          "r"(z[29]), "r"(z[30]), "r"(z[31])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  if (warp >= 1) {
    asm volatile("bar.sync 1, %0;" ::"r"(5 * 32) : "memory");  // MMA warp + epilogue warps
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA
    if (lane == 0) {
      for (int st = 0; st < nstage; ++st) {
        const int s = st % kI8Stages;
        i8_mbar_wait(&empty[s], ((st / kI8Stages) & 1) ^ 1);
        unsigned char* a = base + s * kI8StageBytes;
        unsigned char* b = a + kI8ABytes;
        const unsigned bb = (unsigned)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb),
                     "r"((unsigned)kI8StageBytes)
                     : "memory");
        const int k = (int)(2 * (vs + (size_t)st * kI8StageVox));  // byte of the group's row
        // [plane][rows][128 B]: bytes 0-63 Xr digits, 64-127 Xi digits
        i8_tma3(a, &mapA, k, m0, 0, &full[s]);
        i8_tma3(b, &mapB, k, n0, 0, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    // idesc: D s32 (2 << 4), A s8 (1 << 7), B s8 (1 << 10), K-major, N, M = 128.
    // Per A digit plane d the B planes d' = 1 .. min(4, 6 - d) are consecutive
    // in shared memory (48 rows each) and their levels d + d' are consecutive
    // in TMEM (48 columns each): one MMA with N = 48 (6 - d capped at 4)
    // covers them all -- A is read once per plane instead of once per pair.
    auto idesc_n = [](int n) {
      return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    };
    for (int st = 0; st < nstage; ++st) {
      const int s = st % kI8Stages;
      i8_mbar_wait(&full[s], (st / kI8Stages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t sa = (unsigned)__cvta_generic_to_shared(base + s * kI8StageBytes);
        const uint32_t sb = sa + kI8ABytes;
        // plane p: A at sa + p * 16 KB, B at sb + p * 6 KB; K step ks at +32 ks
        // bytes (ks 0, 1: Xr digits, 2, 3: Xi digits)
#pragma unroll
        for (int d = 1; d <= 4; ++d) {
          const int cnt = (kI8MaxLevel - d) < 4 ? (kI8MaxLevel - d) : 4;  // B planes 1 .. cnt
          const uint32_t idesc = idesc_n(kI8TileN * cnt);
          const uint32_t d_re = tmem + (uint32_t)((d - 1) * kI8TileN);  // level d + 1 onwards
          const uint32_t d_p = tmem + (uint32_t)(256 + (d - 1) * kI8TileN);
          const uint32_t pa = sa + (d - 1) * 16384;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            i8_mma(d_re, i8_desc_sw128(pa + 32 * ks), i8_desc_sw128(sb + 32 * ks), idesc, 1u);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            i8_mma(d_p, i8_desc_sw128(pa + 32 * ks), i8_desc_sw128(sb + 64 + 32 * ks), idesc, 1u);
        }
        i8_commit(&empty[s]);
        if (st == nstage - 1) i8_commit(accfull);
      }
      __syncwarp();
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // Warp w reads TMEM lanes [32 q, 32 q + 32), q = w % 4: A row il.
    const int q = warp & 3;
    const int il = 32 * q + lane;
    const int i = m0 + il;
    double2* out = part + ((size_t)split * g.ntile + tile) * (size_t)kI8TileM * kI8TileN +
                   (size_t)il * kI8TileN;
    if (nstage == 0) {
      if (i < g.F)
        for (int c = 0; c < nn; ++c) out[c] = make_double2(0.0, 0.0);
    } else {
      i8_mbar_wait(accfull, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int ei = i < g.F ? frame_exp(g.amax[i]) : 0;
      for (int c0 = 0; c0 < nn; c0 += 16) {
        double re[16], pp[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) re[u] = pp[u] = 0.0;
#pragma unroll
        for (int lv = 2; lv <= kI8MaxLevel; ++lv) {
          uint32_t r[16], p[16];
          const uint32_t row = (uint32_t)(32 * q) << 16;
          const uint32_t a_re = tmem + row + (uint32_t)((lv - 2) * kI8TileN + c0);
          const uint32_t a_p = tmem + row + (uint32_t)(256 + (lv - 2) * kI8TileN + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15}, [%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
              : "r"(a_re));
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15}, [%16];"
              : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]),
                "=r"(p[6]), "=r"(p[7]), "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]),
                "=r"(p[12]), "=r"(p[13]), "=r"(p[14]), "=r"(p[15])
              : "r"(a_p));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const double w = ldexp(1.0, -7 * lv);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            re[u] += (double)(int)r[u] * w;
            pp[u] += (double)(int)p[u] * w;
          }
        }
        if (i < g.F) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = n0 + c0 + u;
            if (c0 + u < nn && j < g.F) {
              const int e = ei + frame_exp(g.amax[j]);
              out[c0 + u] = make_double2(ldexp(re[u], e), ldexp(pp[u], e));
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// The tile of the list holding (i, j): the first whose rows and columns
// contain it (tiles overlap only in rows computed twice, identically).
FQFG_DEVICE int i8_tile_of(const I8Gram& g, int i, int j) {
  for (int t = 0; t < g.ntile; ++t)
    if (i >= g.m0[t] && i < g.m0[t] + kI8TileM && j >= g.n0[t] && j < g.n0[t] + g.nn[t]) return t;
  return -1;
}

// G[i][j] (+)= sum over splits (fixed order) of Re part[i][j] + i (P[i][j] - P[j][i]).
__global__ void gram_i8_reduce_kernel(const double2* __restrict__ part, const I8Gram g,
                                      double2* __restrict__ G, int accumulate) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)g.F * g.F) return;
  const int i = (int)(idx / g.F), j = (int)(idx % g.F);
  const int t1 = i8_tile_of(g, i, j), t2 = i8_tile_of(g, j, i);
  const size_t o1 = (size_t)(i - g.m0[t1]) * kI8TileN + (j - g.n0[t1]);
  const size_t o2 = (size_t)(j - g.m0[t2]) * kI8TileN + (i - g.n0[t2]);
  const size_t ts = (size_t)kI8TileM * kI8TileN;
  double re = 0.0, im = 0.0;
  for (int s = 0; s < g.nsplit; ++s) {
    const double2 a = part[((size_t)s * g.ntile + t1) * ts + o1];
    const double2 b = part[((size_t)s * g.ntile + t2) * ts + o2];
    re += a.x;
    im += a.y - b.y;
  }
  if (accumulate) {
    re += G[idx].x;
    im += G[idx].y;
  }
  G[idx] = make_double2(re, im);
}

}  // namespace fqfg
