// gram_tc.cu -- Casorati Gram G = X^H X on the 5th-generation tensor cores
// (tcgen05, kind::tf32, accumulators in TMEM), 3xTF32 split for f32-level
// products, FP64 cross-split reduction.
//
// X [F][N] complex64 is read as a real F x 2N matrix R (re/im interleaved
// along K).  With S = R (-i)  (each (re, im) -> (im, -re)):
//     Re G = R R^T,   Im G = R S^T.
// Per K stage (16 voxels = 32 floats = one 128 B swizzle row per frame):
//   warp 0      TMA (cp.async.bulk.tensor, SWIZZLE_128B) of R: all frames x 128 B
//   warps 2-5   split R = hi + lo (hi = R truncated to TF32, written back),
//               S = swapneg(hi), S_lo = swapneg(lo)
//               in shared memory (same swizzled positions), zero voxels outside
//               the split, fence.proxy.async, arrive ready[s]
//   warp 1      one thread issues 6 tcgen05.mma per 8-float K slice:
//               D_re += A R^T + A R_lo^T + A_lo R^T, D_im likewise with S
//               (A = the M-tile's rows of R), then tcgen05.commit -> empty[s]
//   warps 6-9   epilogue: after every chunk of g.chunk stages, tcgen05.ld the
//               fp32 accumulators (TMEM -> registers), add them (red.add, round
//               to nearest) into this CTA's running fp32 partial in global
//               memory (column-major, coalesced, L2-resident), release TMEM.
// The tensor core's fp32 accumulation truncates (measured ~5e-8 relative per
// accumulation, a bias that grows linearly with the accumulation count), so
// the TMEM accumulator is restarted every chunk (g.chunk x 12 accumulations)
// and chunks are summed with round-to-nearest adds.  Each CTA walks a
// contiguous super-split of voxels; gram_tc_reduce sums the CTAs' partials in
// FP64 in a fixed order (deterministic).  Only the upper triangle is formed:
// M-tile t covers rows [r0, r0 + 128) and columns j >= r0.
#include <cuda.h>

#include "common.cuh"

namespace fqfg {

constexpr int kTcThreads = 320;
constexpr int kTcStages = 2;

struct TcGram {
  int F, Fp, rows;   // frames, frames padded to 16, tile rows (max(Fp, 128))
  int nmt;           // M tiles
  int nsplit;        // super-splits (CTAs per M tile)
  int chunk;         // stages (16 voxels each) per TMEM accumulation
  size_t stages_per_split;
  size_t N, v0, v1;  // voxel count, range
};

FQFG_DEVICE int tc_row0(const TcGram& g, int mt) { return min(128 * mt, g.rows - 128); }

FQFG_DEVICE uint64_t umma_desc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B: LBO = 1 (unused), SBO = 1024 B (8 rows x 128 B),
  // version 1 (sm_100), layout type 2 (SWIZZLE_128B).
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

FQFG_DEVICE void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

FQFG_DEVICE void tc_commit(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a)
               : "memory");
}

FQFG_DEVICE uint32_t tf32_idesc(int n) {
  // c_format F32 (bit 4), a/b format TF32 (2 at bits 7 and 10), K-major A/B,
  // N >> 3 at bit 17, M >> 4 at bit 24 (M = 128).
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    gram_tc_kernel(const __grid_constant__ CUtensorMap tmap, const TcGram g,
                   float* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 1024-B aligned operand buffers: [stage][R, R_lo, S, S_lo][rows][128 B]
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int buf_bytes = g.rows * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kTcStages * 4 * buf_bytes);
  uint64_t* full = bars;                    // [stages] TMA landed
  uint64_t* ready = bars + kTcStages;       // [stages] derived tiles written
  uint64_t* empty = bars + 2 * kTcStages;   // [stages] MMAs done reading
  uint64_t* accfull = bars + 3 * kTcStages;  // chunk accumulated (tcgen05.commit)
  uint64_t* accempty = accfull + 1;           // chunk drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x % g.nmt, split = blockIdx.x / g.nmt;
  const size_t vs = min(g.v1, g.v0 + (size_t)split * g.stages_per_split * 16);
  const size_t ve = min(g.v1, vs + g.stages_per_split * 16);
  // TMA box starts must be 16-B aligned: stages start at the even voxel vb
  // <= vs; the transform zeroes voxels outside [vs, ve).
  const size_t vb = vs & ~(size_t)1;
  const int nstage = ve > vs ? (int)((ve - vb + 15) / 16) : 0;
  const int nchunk = (nstage + g.chunk - 1) / g.chunk;
  const int r0 = tc_row0(g, mt);
  const int ncol = g.Fp - r0;  // columns j >= r0 (multiple of 16)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accfull, 1);
    mbar_init(accempty, 4);
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA
    if (lane == 0) {
      for (int st = 0; st < nstage; ++st) {
        const int s = st % kTcStages;
        mbar_wait(&empty[s], ((st / kTcStages) & 1) ^ 1);
        unsigned char* dst = base + s * 4 * buf_bytes;
        mbar_expect_tx(&full[s], (unsigned)buf_bytes);
        const int c0 = (int)(2 * (vb + 16 * (size_t)st));
        unsigned d = (unsigned)__cvta_generic_to_shared(dst);
        unsigned b = (unsigned)__cvta_generic_to_shared(&full[s]);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3}], [%4];" ::"r"(d),
            "l"(&tmap), "r"(c0), "r"(0), "r"(b)
            : "memory");
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA
    const uint32_t id = tf32_idesc(ncol);
    const uint32_t d_re = tmem, d_im = tmem + (uint32_t)ncol;
    for (int st = 0; st < nstage; ++st) {
      const int s = st % kTcStages;
      const int c = st / g.chunk;
      const bool first = st % g.chunk == 0;
      if (first && c > 0) mbar_wait(accempty, (c - 1) & 1);  // TMEM drained
      mbar_wait(&ready[s], (st / kTcStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t sb = (unsigned)__cvta_generic_to_shared(base + s * 4 * buf_bytes);
        const uint32_t off = (uint32_t)r0 * 128;
        const uint32_t R = sb + off, Rl = sb + buf_bytes + off, S = sb + 2 * buf_bytes + off,
                       Sl = sb + 3 * buf_bytes + off;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t ko = 32 * k;
          const uint64_t a = umma_desc_sw128(R + ko), al = umma_desc_sw128(Rl + ko);
          const uint64_t b = umma_desc_sw128(R + ko), bl = umma_desc_sw128(Rl + ko);
          const uint64_t cc = umma_desc_sw128(S + ko), cl = umma_desc_sw128(Sl + ko);
          const uint32_t acc = (!first || k > 0) ? 1u : 0u;
          tc_mma(d_re, a, b, id, acc);
          tc_mma(d_re, a, bl, id, 1u);
          tc_mma(d_re, al, b, id, 1u);
          tc_mma(d_im, a, cc, id, acc);
          tc_mma(d_im, a, cl, id, 1u);
          tc_mma(d_im, al, cc, id, 1u);
        }
        tc_commit(&empty[s]);
        if (st % g.chunk == g.chunk - 1 || st == nstage - 1) tc_commit(accfull);
      }
      __syncwarp();
    }
  } else if (warp < 6) {
    // ----------------------------------------------------------- transform
    const int t = threadIdx.x - 64;  // 0..127
    const int nch = g.rows * 8;
    for (int st = 0; st < nstage; ++st) {
      const int s = st % kTcStages;
      mbar_wait(&full[s], (st / kTcStages) & 1);
      float4* R = reinterpret_cast<float4*>(base + s * 4 * buf_bytes);
      float4* Rl = R + buf_bytes / 16;
      float4* S = R + 2 * buf_bytes / 16;
      float4* Sl = R + 3 * buf_bytes / 16;
      const size_t vst = vb + 16 * (size_t)st;
      for (int c = t; c < nch; c += 128) {
        const int row = c >> 3, phys = c & 7, logical = phys ^ (row & 7);
        const size_t vox = vst + 2 * logical;  // this chunk: voxels vox, vox + 1
        float4 x = R[c];
        if (vox >= ve || vox < vs) x.x = x.y = 0.f;
        if (vox + 1 >= ve || vox + 1 < vs) x.z = x.w = 0.f;
        // hi = x truncated to TF32 (written back, so the tensor core sees an
        // exactly representable value whatever its f32 -> tf32 conversion),
        // lo = x - hi exactly.
        float4 hi, lo;
        hi.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
        hi.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
        hi.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
        hi.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
        lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
        R[c] = hi;
        Rl[c] = lo;
        S[c] = make_float4(hi.y, -hi.x, hi.w, -hi.z);
        Sl[c] = make_float4(lo.y, -lo.x, lo.w, -lo.z);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&ready[s]);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Warp w reads TMEM lanes [32 q, 32 q + 32), q = w % 4, i.e. row il of the
    // M tile; the CTA's partial is column-major [2 Fp][128] so a warp's 32
    // lanes touch 128 contiguous bytes per column.
    const int q = warp & 3;
    const int il = 32 * q + lane;
    float* out = part + (size_t)(split * g.nmt + mt) * (2 * g.Fp) * 128 + il;
    for (int c = 0; c < nchunk; ++c) {
      mbar_wait(accfull, c & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int col = 0; col < 2 * ncol; col += 16) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)col;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // The partial is private to this thread: first chunk stores, later
        // chunks issue fire-and-forget reductions (round to nearest; same
        // thread, same address -> program order, deterministic).
        if (c == 0) {
#pragma unroll
          for (int u = 0; u < 16; ++u) out[(size_t)(col + u) * 128] = __uint_as_float(r[u]);
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(out + (size_t)(col + u) * 128),
                         "f"(__uint_as_float(r[u]))
                         : "memory");
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty);
    }
    if (nchunk == 0) {  // empty split: zero partial
      for (int col = 0; col < 2 * ncol; ++col) out[(size_t)col * 128] = 0.f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// G[i][j] = sum over splits (FP64, split order) of the partial of the M tile
// that owns row i with column j >= its r0; lower triangle by Hermitian mirror.
__global__ void gram_tc_reduce(const float* __restrict__ part, const TcGram g,
                               double2* __restrict__ G, int accumulate) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)g.F * g.F) return;
  int i = (int)(idx / g.F), j = (int)(idx % g.F);
  const bool mirror = i > j;
  const int a = mirror ? j : i, b = mirror ? i : j;
  int mt = 0;
  for (int t = 0; t < g.nmt; ++t)
    if (tc_row0(g, t) <= a) mt = t;
  const int r0 = tc_row0(g, mt), ncol = g.Fp - r0, il = a - r0;
  double re = 0.0, im = 0.0;
  for (int s = 0; s < g.nsplit; ++s) {
    const float* p = part + (size_t)(s * g.nmt + mt) * (2 * g.Fp) * 128 + il;
    re += (double)p[(size_t)(b - r0) * 128];
    im += (double)p[(size_t)(ncol + (b - r0)) * 128];
  }
  if (mirror) im = -im;
  if (i == j) im = 0.0;
  if (accumulate) {
    re += G[idx].x;
    im += G[idx].y;
  }
  G[idx] = make_double2(re, im);
}

}  // namespace fqfg
