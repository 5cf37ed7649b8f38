// das_tc.cu -- delay-and-sum on the 5th-generation tensor cores (opt-in,
// FQFG_DAS_KERNEL=3).
//
// For one (element, angle) and a tile of 64 voxels the interpolated,
// carrier-rotated sum over the two taps is a dense product with a sparse
// weight matrix:
//     out[v][f] += sum_k W[v][k] X[k][f],   k = (time row, re/im)
// W has four nonzeros per (voxel, re/im) row:  c (1 - frac), c frac at the
// rows s0, s0 + 1 (das.cpp:182-197, e^{+i 2 pi f_c tau}), written as the real
// 2x2 block [[Wr, -Wi], [Wi, Wr]] so that re and im of the output are rows
// m = v and m = 64 + v of one M = 128 MMA.  X is the element's IQ window:
// rows [t_base, t_base + 8 nb) x all frames of the pass, N = fpass.
//
// Precision: X and W are split into fp16 hi + lo (x S = hi + lo, S a power of
// two from max |RF| so |x S| <= 6e4), three MMAs per K block
// (hi.hi + hi.lo + lo.hi, each kind::f16 with fp32 accumulation), so the
// product error is ~2^-22 relative.  The tensor core's fp32 accumulation
// truncates (~5e-8 per accumulation, biased), so the TMEM accumulator is
// restarted every kTcChunk stages and drained into fp32 registers with
// round-to-nearest adds (double-buffered: 2 x fpass TMEM columns).
//
// Roles (416 threads):
//   warps 0-3   producers: FP64 reference-exact delay table (same code path as
//               das2), conservative window of the tile box -> TMA of X boxes
//               (16 fp16 x fpass, SWIZZLE_32B) issued before the table, then W
//               rows in the same SWIZZLE_32B K-major layout; one arrival on
//               full[slot] with the TMA bytes.
//   warp 4      TMEM allocation; one thread issues 3 nb tcgen05.mma per stage,
//               commits empty[slot] and, per chunk, accfull[buffer].
//   warps 5-12  epilogue: tcgen05.ld of the finished chunk (quadrant w % 4,
//               column half (w - 5) / 4: 104 fp32 per thread), add, release.
// Layouts: IQ16[plane][a][e][frame][TP][re, im] fp16 (time innermost, TP =
// T rounded to 4 so the row pitch is 16 B aligned); the TMA's out-of-range
// zero fill supplies the t = -1 and t = T guard rows.
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace fqfg {

constexpr int kTcV = 64;       // voxels per tile
constexpr int kTcNB = 2;       // max K blocks (8 time rows) per stage; wider windows -> parts
constexpr int kTcSlots = 3;    // operand pipeline depth
constexpr int kTcChunk = 16;   // stages per TMEM accumulation (16: 7e-6 max rel. error)
constexpr int kTcProd = 128;   // producer threads
constexpr int kTcEB = 4;       // elements per producer block (EB x A <= kTcTab)
constexpr int kTcTab = 36;     // table capacity in (element, angle) pairs of 64 voxels
constexpr int kTcDasThreads = 416;
constexpr int kTcXBox = 7168;  // one X box (fpass <= 224 rows x 32 B), 1 KB aligned

struct TcSlotHdr {
  int done, nb, t_base, pad;
};

// Shared-memory carve-up (bytes from a 1 KB aligned base).
struct TcSmem {
  static constexpr int x_off = 0;                                          // [S][NB][2] X boxes
  static constexpr int w_off = x_off + kTcSlots * kTcNB * 2 * kTcXBox;      // [S][NB][2] W 4 KB
  static constexpr int tab_off = w_off + kTcSlots * kTcNB * 2 * 4096;       // [EB][A][64] float4
  static constexpr int rc_off = tab_off + kTcTab * kTcV * 16;              // [EB][64] double
  static constexpr int vox_off = rc_off + kTcEB * kTcV * 8;                // [64][3] double
  static constexpr int ttx_off = vox_off + kTcV * 24;                      // [A <= 16][64] double
  static constexpr int tb_off = ttx_off + 16 * kTcV * 8;                   // [A][2] double
  static constexpr int db_off = tb_off + 16 * 16;                          // [EB][2] double
  static constexpr int hdr_off = db_off + kTcEB * 16;                      // [S] TcSlotHdr
  static constexpr int bar_off = hdr_off + 64;                             // barriers
  static constexpr int total = bar_off + 16 * 8 + 64;
};
constexpr size_t das_tc_smem() { return TcSmem::total + 1024; }

FQFG_DEVICE uint64_t umma_desc_sw32(uint32_t saddr) {
  // K-major SWIZZLE_32B: rows of 32 B, 8-row atoms of 256 B (SBO), version 1,
  // layout type 6.
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}

FQFG_DEVICE void tc_mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

FQFG_DEVICE uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

__global__ void __launch_bounds__(kTcDasThreads, 1)
    das_tc_kernel(const DasParams p, const DasLaunch L, const __grid_constant__ CUtensorMap tmap,
                  const float* __restrict__ d_scale, float2* __restrict__ x,
                  unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 1 KB aligned base, derived from smem_raw so the compiler keeps the
  // shared address space (LDS/STS, not generic loads)
  unsigned char* base =
      smem_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  unsigned char* xs = base + TcSmem::x_off;
  unsigned char* ws = base + TcSmem::w_off;
  float4* tab = reinterpret_cast<float4*>(base + TcSmem::tab_off);
  double* rc = reinterpret_cast<double*>(base + TcSmem::rc_off);
  double* vox = reinterpret_cast<double*>(base + TcSmem::vox_off);
  double* ttxA = reinterpret_cast<double*>(base + TcSmem::ttx_off);
  double* tbound = reinterpret_cast<double*>(base + TcSmem::tb_off);
  double* dbound = reinterpret_cast<double*>(base + TcSmem::db_off);
  TcSlotHdr* hdr = reinterpret_cast<TcSlotHdr*>(base + TcSmem::hdr_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + TcSmem::bar_off);  // [S]
  uint64_t* empty = full + kTcSlots;                                      // [S]
  uint64_t* accfull = full + 2 * kTcSlots;                                // [2]
  uint64_t* accempty = accfull + 2;                                       // [2]
  int* misc = reinterpret_cast<int*>(accempty + 2);  // [0] tmem, [1] active bits, [2..3] n, [4..5] final

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fpass = p.fpass;
  int tile = blockIdx.x;
  const int tx = tile % L.tiles_x;
  tile /= L.tiles_x;
  const int ty = tile % L.tiles_y;
  const int tz = tile / L.tiles_y;
  const int i0 = tx * L.TX, j0 = ty * L.TY, k0 = L.kbeg + tz * L.TZ;

  for (int l = tid; l < kTcV; l += blockDim.x) {
    const int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
    const int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    const bool ok = i < p.nx && j < p.ny && k < L.kend;
    vox[3 * l] = ok ? grid_coord(p.ox, i, p.sx) : __longlong_as_double(0x7ff8000000000000ll);
    vox[3 * l + 1] = grid_coord(p.oy, j, p.sy);
    vox[3 * l + 2] = grid_coord(p.oz, k, p.sz);
  }
  if (tid == 0) {
    for (int s = 0; s < kTcSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&accfull[s], 2);
      mbar_init(&accempty[s], 8);
    }
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 4) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(misc);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = (uint32_t)misc[0];
  for (int i = tid; i < p.A * kTcV; i += blockDim.x) {
    const int a = i / kTcV, l = i % kTcV;
    const AngleConst ac = p.ang[a];
    ttxA[i] = tx_delay(vox[3 * l], vox[3 * l + 2], ac.sina, ac.cosa, ac.ref, p.c);
  }
  __syncthreads();

  if (warp < 4) {
    // ============================ producers ============================
    const int tp = tid;
    unsigned long long n_oow = 0, n_taps = 0;
    int stage = 0;
    const int EB = min(kTcEB, kTcTab / p.A);
    const int AV = p.A * kTcV;
    const int i1 = min(i0 + L.TX, p.nx) - 1, j1 = min(j0 + L.TY, p.ny) - 1,
              k1 = min(k0 + L.TZ, L.kend) - 1;
    const double bx0 = grid_coord(p.ox, i0, p.sx), bx1 = grid_coord(p.ox, i1, p.sx);
    const double by0 = grid_coord(p.oy, j0, p.sy), by1 = grid_coord(p.oy, j1, p.sy);
    const double bz0 = grid_coord(p.oz, k0, p.sz), bz1 = grid_coord(p.oz, k1, p.sz);
    for (int a = tp; a < p.A; a += kTcProd) {
      const AngleConst ac = p.ang[a];
      tbound[2 * a] = (fmin(bx0 * ac.sina, bx1 * ac.sina) + bz0 * ac.cosa - ac.ref) / p.c;
      tbound[2 * a + 1] = (fmax(bx0 * ac.sina, bx1 * ac.sina) + bz1 * ac.cosa - ac.ref) / p.c;
    }
    const long long plane_rows = (long long)p.A * p.E * fpass;
    for (int e0 = 0; e0 < p.E; e0 += EB) {
      const int neb = min(EB, p.E - e0);
      if (tp == 0) misc[1] = 0;
      named_sync(1, kTcProd);
      // (1) receive delays / aperture of EB elements x 64 voxels; per-element
      //     receive-range bounds over the tile box
      for (int idx = tp; idx < kTcEB * kTcV; idx += kTcProd) {
        const int el = idx / kTcV, v = idx % kTcV, e = e0 + el;
        double r = -1.0;
        const double px = vox[3 * v], py = vox[3 * v + 1], pz = vox[3 * v + 2];
        if (el < neb && px == px) {
          const double ex = __ldg(p.elem + 3 * e), ey = __ldg(p.elem + 3 * e + 1),
                       ez = __ldg(p.elem + 3 * e + 2);
          if (!(p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum)))
            r = rx_delay(px, py, pz, ex, ey, ez, p.c);
        }
        rc[idx] = r;
        const unsigned bits = __reduce_or_sync(0xffffffffu, r >= 0.0 ? 1u << el : 0u);
        if (lane == 0 && bits) atomicOr(&misc[1], (int)bits);
      }
      if (tp < neb) {
        const int e = e0 + tp;
        const double ex = __ldg(p.elem + 3 * e), ey = __ldg(p.elem + 3 * e + 1),
                     ez = __ldg(p.elem + 3 * e + 2);
        const double dxn = fmax(fmax(bx0 - ex, ex - bx1), 0.0);
        const double dyn = fmax(fmax(by0 - ey, ey - by1), 0.0);
        const double dzn = fmax(fmax(bz0 - ez, ez - bz1), 0.0);
        const double dxf = fmax(fabs(bx0 - ex), fabs(bx1 - ex));
        const double dyf = fmax(fabs(by0 - ey), fabs(by1 - ey));
        const double dzf = fmax(fabs(bz0 - ez), fabs(bz1 - ez));
        dbound[2 * tp] = sqrt(dxn * dxn + dyn * dyn + dzn * dzn) / p.c;
        dbound[2 * tp + 1] = sqrt(dxf * dxf + dyf * dyf + dzf * dzf) / p.c;
      }
      named_sync(1, kTcProd);
      const int active = misc[1];
      if (!active) continue;
      // (2) exact table of every (element, angle, voxel) (das.cpp:159-197,
      //     as das2's producer), many independent entries per thread
      for (int idx = tp; idx < neb * AV; idx += kTcProd) {
        const int el = idx / AV, rem = idx % AV, v = rem % kTcV;
        const double r = rc[el * kTcV + v];
        float4 ent = make_float4(__int_as_float(kInactive), 0.f, 0.f, 0.f);
        if (r >= 0.0) {
          const AngleConst ac = p.ang[rem / kTcV];
          const double tau = xadd(ttxA[rem], r);
          const double sv = xmul(xsub(tau, ac.t0), p.fs);
          int s0 = kInactive;
          float frac = 0.f;
          if (p.interp) {
            const double sfl = floor(sv);
            const double fr = xsub(sv, sfl);
            const bool live0 = sfl >= 0.0 && sfl < (double)p.T;
            const bool live1 = fr > 0.0 && xadd(sfl, 1.0) >= 0.0 && xadd(sfl, 1.0) < (double)p.T;
            if (live0 || live1) {
              s0 = (int)sfl;
              frac = (float)fr;
              n_taps += (int)live0 + (int)live1;
            } else {
              ++n_oow;
            }
          } else {
            const double ri = round(sv);
            if (ri >= 0.0 && ri < (double)p.T) {
              s0 = (int)ri;
              ++n_taps;
            } else {
              ++n_oow;
            }
          }
          if (s0 != kInactive) {
            double cyc = p.fc * tau;
            cyc -= rint(cyc);
            float sn, cs;
            sincospif(2.0f * (float)cyc, &sn, &cs);
            ent = make_float4(__int_as_float(s0), frac, cs, sn);
          }
        }
        tab[idx] = ent;
      }
      named_sync(1, kTcProd);

      // (3) one stage per (element, angle, window part)
      for (int el = 0; el < neb; ++el) {
        if (!((active >> el) & 1)) continue;
        const int e = e0 + el;
        for (int a = 0; a < p.A; ++a) {
          const AngleConst ac = p.ang[a];
          // Conservative rows of the taps over the tile box (one row of
          // margin, as das2); the TMA box start must be 16-B aligned (4 time
          // rows of fp16 re/im), so the window starts at lo & ~3.
          const double smin = (tbound[2 * a] + dbound[2 * el] - ac.t0) * p.fs;
          const double smax = (tbound[2 * a + 1] + dbound[2 * el + 1] - ac.t0) * p.fs;
          const double flo = fmax(floor(smin) - 1.0, -1.0);
          const double fhi = fmin(floor(smax) + 1.0, (double)(p.T - 1));
          if (flo > fhi) continue;  // every tap out of window (counted in the table)
          const int lo = (int)flo & ~3, n = (int)fhi + 2 - lo;
          // parts of <= 8 NB rows overlapping by four (a tap pair never
          // straddles two parts; every part base stays 4-row aligned)
          const int span = 8 * kTcNB - 4;
          const int nparts = n <= 8 * kTcNB ? 1 : 1 + (n - 8 * kTcNB + span - 1) / span;
          const long long row_ae = ((long long)a * p.E + e) * fpass;
          const float4 ent = tab[(el * p.A + a) * kTcV + (tp & 63)];
          for (int part = 0; part < nparts; ++part) {
            const int slot = stage % kTcSlots;
            mbar_wait(&empty[slot], ((stage / kTcSlots) & 1) ^ 1);
            const int t_base = lo + part * span;
            const int rows = min(8 * kTcNB, lo + n - t_base);
            const int nb = (rows + 7) / 8;
            if (tp == 0) {
              hdr[slot].done = 0;
              hdr[slot].nb = nb;
              hdr[slot].t_base = t_base;
              if (!(L.debug & 0x20000)) {
                const unsigned bytes = (unsigned)(nb * 2 * fpass * 32);
                const unsigned bb = (unsigned)__cvta_generic_to_shared(&full[slot]);
                asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bb), "r"(bytes)
                             : "memory");
                for (int kb = 0; kb < nb; ++kb)
                  for (int pl = 0; pl < 2; ++pl) {
                    const unsigned d = (unsigned)__cvta_generic_to_shared(
                        xs + ((slot * kTcNB + kb) * 2 + pl) * kTcXBox);
                    const int c0 = 2 * t_base + 16 * kb;
                    const int c1 = (int)(pl * plane_rows + row_ae);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::"
                        "bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(d),
                        "l"(&tmap), "r"(c0), "r"(c1), "r"(bb)
                        : "memory");
                  }
              }
            }
            // W row m = tp (voxel m & 63; re for m < 64, im else), whole row in
            // registers: words (one time row's re/im pair each) r0 and r0 + 1
            // carry the tap weights, all others zero.
            {
              const int m = tp, c = m >> 6;
              const int s0 = __float_as_int(ent.x);
              const int r0 = s0 - t_base;
              const bool act = s0 != kInactive && r0 >= 0 && r0 + 1 < 8 * kTcNB &&
                               (part + 1 == nparts || r0 < span);
              const float fr = ent.y, cr = ent.z, ci = ent.w;
              const float w0 = 1.0f - fr;
              // k = 2 row + (re, im): re row Wr0, -Wi0 | Wr1, -Wi1 ; im row Wi0, Wr0 | Wi1, Wr1
              const float q0 = c ? ci * w0 : cr * w0, q1 = c ? cr * w0 : -(ci * w0);
              const float q2 = c ? ci * fr : cr * fr, q3 = c ? cr * fr : -(ci * fr);
              const __half2 h01 = __floats2half2_rn(q0, q1), h23 = __floats2half2_rn(q2, q3);
              const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
              const uint32_t H0 = act ? h2u(h01) : 0u, H1 = act ? h2u(h23) : 0u;
              const uint32_t L0 = act ? h2u(__floats2half2_rn(q0 - f01.x, q1 - f01.y)) : 0u;
              const uint32_t L1 = act ? h2u(__floats2half2_rn(q2 - f23.x, q3 - f23.y)) : 0u;
              unsigned char* wrow = ws + slot * kTcNB * 2 * 4096 + m * 32;
              const int sw = (m >> 2) & 1;
              for (int kb = 0; kb < nb; ++kb) {
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                  const int j0w = 8 * kb + 4 * ch;  // first word (time row) of the chunk
                  uint32_t hv[4], lv[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    const int d = j0w + u - r0;
                    hv[u] = d == 0 ? H0 : d == 1 ? H1 : 0u;
                    lv[u] = d == 0 ? L0 : d == 1 ? L1 : 0u;
                  }
                  const int off = kb * 2 * 4096 + ((ch ^ sw) << 4);
                  *reinterpret_cast<uint4*>(wrow + off) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
                  *reinterpret_cast<uint4*>(wrow + off + 4096) =
                      make_uint4(lv[0], lv[1], lv[2], lv[3]);
                }
              }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_sync(1, kTcProd);
            if (tp == 0) mbar_arrive(&full[slot]);
            ++stage;
          }
        }
      }
    }
    // termination stage
    const int slot = stage % kTcSlots;
    mbar_wait(&empty[slot], ((stage / kTcSlots) & 1) ^ 1);
    if (tp == 0) {
      hdr[slot].done = 1;
      mbar_arrive(&full[slot]);
    }
    if (counters && L.pass == 0) {
      for (int o = 16; o > 0; o >>= 1) {
        n_oow += __shfl_xor_sync(0xffffffffu, n_oow, o);
        n_taps += __shfl_xor_sync(0xffffffffu, n_taps, o);
      }
      if (lane == 0) {
        atomicAdd(counters, n_oow);
        atomicAdd(counters + 1, n_taps);
      }
    }
  } else if (warp == 4) {
    // ============================== MMA ==============================
    const uint32_t idesc = (1u << 4) | ((uint32_t)(fpass >> 3) << 17) | ((128u >> 4) << 24);
    int chunk = 0, in_chunk = 0;
    const int chunk_len = L.pf > 0 ? L.pf : kTcChunk;  // (experiments: FQFG_DAS_PF)
    for (int stage = 0;; ++stage) {
      const int slot = stage % kTcSlots;
      mbar_wait(&full[slot], (stage / kTcSlots) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const TcSlotHdr h = hdr[slot];
      const int b = chunk & 1;
      if (h.done) {
        if (lane == 0) {
          misc[2 + b] = in_chunk;
          misc[4 + b] = 1;
          tc_commit(&accfull[b]);
          mbar_arrive(&accfull[b]);
        }
        __syncwarp();
        break;
      }
      if (in_chunk == 0 && chunk >= 2) mbar_wait(&accempty[b], ((chunk >> 1) - 1) & 1);
      if (lane == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(256 * b);
        const uint32_t xb =
            (uint32_t)__cvta_generic_to_shared(xs + slot * kTcNB * 2 * kTcXBox);
        const uint32_t wb = (uint32_t)__cvta_generic_to_shared(ws + slot * kTcNB * 2 * 4096);
        for (int kb = 0; kb < h.nb; ++kb) {
          const uint64_t wh = umma_desc_sw32(wb + (kb * 2 + 0) * 4096);
          const uint64_t wl = umma_desc_sw32(wb + (kb * 2 + 1) * 4096);
          const uint64_t xh = umma_desc_sw32(xb + (kb * 2 + 0) * kTcXBox);
          const uint64_t xl = umma_desc_sw32(xb + (kb * 2 + 1) * kTcXBox);
          if (L.debug & 0x10000) continue;  // diagnostic: no MMAs
          tc_mma_f16(d, wh, xh, idesc, (in_chunk > 0 || kb > 0) ? 1u : 0u);
          tc_mma_f16(d, wh, xl, idesc, 1u);
          tc_mma_f16(d, wl, xh, idesc, 1u);
        }
        tc_commit(&empty[slot]);
      }
      __syncwarp();
      if (++in_chunk == chunk_len) {
        if (lane == 0) {
          misc[2 + b] = in_chunk;
          misc[4 + b] = 0;
          tc_commit(&accfull[b]);
          mbar_arrive(&accfull[b]);
        }
        __syncwarp();
        in_chunk = 0;
        ++chunk;
      }
    }
  } else {
    // ============================ epilogue ============================
    const int q = warp & 3, half = (warp - 5) >> 2;
    const int m = 32 * q + lane;
    const int ncol = fpass / 2;  // columns of this thread (fpass <= 208: <= 104)
    float acc[104];
#pragma unroll
    for (int j = 0; j < 104; ++j) acc[j] = 0.f;
    for (int chunk = 0;; ++chunk) {
      const int b = chunk & 1;
      mbar_wait_hint(&accfull[b], (chunk >> 1) & 1, 1000000);  // sleep, leave issue slots
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int nst = misc[2 + b], fin = misc[4 + b];
      if (nst > 0 && !(L.debug & 0x40000)) {  // (diagnostic: no TMEM loads)
        const uint32_t taddr =
            tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(256 * b + half * ncol);
#pragma unroll
        for (int g = 0; g < 13; ++g) {
          if (8 * g < ncol) {
            uint32_t r[8];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7])
                : "r"(taddr + 8 * g));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[8 * g + u] += __uint_as_float(r[u]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[b]);
      if (fin) break;
    }
    // out[f][voxel] (re for m < 64, im for m >= 64), x 1 / (A S)
    const int v = m & 63, c = m >> 6;
    const int lx = v % L.TX, ly = (v / L.TX) % L.TY, lz = v / (L.TX * L.TY);
    const int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    if (i < p.nx && j < p.ny && k < L.kend) {
      const float inv = (float)(1.0 / p.A) / __ldg(d_scale);
      const size_t N = (size_t)p.nx * p.ny * p.nz;
      const size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
      float* xo = reinterpret_cast<float*>(x);
#pragma unroll
      for (int jj = 0; jj < 104; ++jj) {
        const int f = L.pass * fpass + half * ncol + jj;
        if (jj < ncol && f < p.F) xo[2 * ((size_t)f * N + flat) + c] = acc[jj] * inv;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// max |RF| over rows [t0, t1] of every (frame, angle) slice -> scale S (a
// power of two with 2 sum|h| max|RF| S <= 6e4, the fp16 range of the IQ
// split).  One block per 64 K floats, atomicMax on the float's bits.
__global__ void rf_absmax_kernel(const float* __restrict__ rf, size_t slices, int T, int E, int t0,
                                 int t1, unsigned* __restrict__ mx) {
  const size_t rows = (size_t)(t1 - t0 + 1) * E;
  const size_t n = slices * rows;
  float m = 0.f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t sl = i / rows, r = i % rows;
    const float v = fabsf(rf[sl * (size_t)T * E + (size_t)t0 * E + r]);
    m = v == v ? fmaxf(m, v) : m;
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, __float_as_uint(m));
}

__global__ void tc_scale_kernel(const unsigned* __restrict__ mx, float hsum, float* __restrict__ s) {
  const float bound = 2.f * hsum * __uint_as_float(*mx);
  float sc = 1.f;
  if (bound > 0.f && isfinite(bound)) {
    const float e = floorf(log2f(6.0e4f / bound));
    sc = exp2f(fminf(fmaxf(e, -100.f), 100.f));
  }
  *s = sc;
}

// Staging [nf][A][T][E] float2 -> IQ16[plane][a][e][frame][TP][2] fp16 (x S,
// hi / lo split); frames >= nf are zeros.  grid (ceil(T/32), ceil(E/32),
// fpass * A); block 256.  Rows outside [t_lo, t_hi] (not demodulated for a
// depth slab) are zeros.
__global__ void __launch_bounds__(256) demod_pack16_kernel(const float2* __restrict__ stage,
                                                           __half* __restrict__ dst,
                                                           const float* __restrict__ d_scale,
                                                           int T, int TP, int E, int A, int nf,
                                                           int fpass, int t_lo, int t_hi) {
  __shared__ float2 tile[32][33];
  const int t0 = blockIdx.x * 32, e0 = blockIdx.y * 32;
  const int f = blockIdx.z / A, a = blockIdx.z % A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float S = __ldg(d_scale);
  for (int r = warp; r < 32; r += 8) {
    const int t = t0 + r, e = e0 + lane;
    float2 v = make_float2(0.f, 0.f);
    // rows outside [t_lo, t_hi] were not demodulated for this slab: zeros
    if (f < nf && t >= t_lo && t <= t_hi && e < E) v = stage[(((size_t)f * A + a) * T + t) * E + e];
    tile[r][lane] = v;
  }
  __syncthreads();
  const size_t plane = (size_t)A * E * fpass * TP * 2;
  for (int el = warp; el < 32; el += 8) {
    const int e = e0 + el, t = t0 + lane;
    if (e >= E || t >= T) continue;
    const float2 v = tile[lane][el];
    const float xr = v.x * S, xi = v.y * S;
    const __half hr = __float2half_rn(xr), hi_ = __float2half_rn(xi);
    const __half lr = __float2half_rn(xr - __half2float(hr)),
                 li = __float2half_rn(xi - __half2float(hi_));
    const size_t o = ((((size_t)a * E + e) * fpass + f) * TP + t) * 2;
    *reinterpret_cast<__half2*>(dst + o) = __halves2half2(hr, hi_);
    *reinterpret_cast<__half2*>(dst + plane + o) = __halves2half2(lr, li);
  }
}

}  // namespace fqfg
