// das_tc.cu -- delay-and-sum on the 5th-generation tensor cores: tcgen05.mma
// with the weight operand in TMEM and the IQ windows in shared memory.
//
// For one (element, angle) and a tile of 64 voxels the interpolated,
// carrier-rotated two-tap sum (das.cpp:309-326) is a dense product with a
// sparse weight matrix:
//     out[m][f] += sum_k W[m][k] X[k][f]
//   m = (re | im output, voxel): 128 rows = one M = 128 MMA,
//   k = (time row, re | im): 8 time rows = K = 16 per MMA ("K block"),
//   f = frames of the pass (N = fpass <= 208).
// W has four nonzeros per row, the real 2x2 form of the complex weights
// c (1 - frac), c frac at the rows s0, s0 + 1 (c = e^{+i 2 pi f_c tau}).
//
// Precision: X (IQ, scaled per frame by a power of two S_f so that
// |x S_f| <= 6e4) and W are split into fp16 hi + lo; three kind::f16 MMAs
// per K block (hi.hi + hi.lo + lo.hi) give ~2^-22 relative products.  The
// tensor core's fp32 accumulation truncates, so the TMEM accumulator is
// restarted every kTcChunk stages and drained into fp32 registers with
// round-to-nearest adds (double-buffered accumulators).
//
// Roles (20 warps, one CTA per SM; warp w issues on sub-partition w % 4, and
// the emitter, the MMA warp and each W writer sit on different ones or share
// one with a single table warp -- measured 2 % (C) / 5 % (B) faster than the
// emitter, MMA warp and W writer 0 together on sub-partition 0):
//   warps 2-3,  table: thread = (element, voxel) of a 3-element block: FP64
//   8-11        reference-exact receive delay / aperture, then tap index,
//               weight and rotation for every angle (das.cpp:159-197, the
//               das2 arithmetic) into 2-4 table buffers; exact tap-row
//               windows per (element, angle) by warp min / max; one warp
//               compacts the windows with taps into the block's list.
//   warp 0      emitter: per listed window, parts of <= 16 rows every 12
//               (a tap pair never straddles two), stage header, the window's
//               4-row chunks of both planes by bulk copy (cp.async.bulk) into
//               an X slot -> xfull.
//   warps 4-7   W writers: lane quadrant w - 4 of the stage's W slot in TMEM
//               (tcgen05.st of 16 columns per K block) -> wfull.
//   warp 1      one elected thread issues 3 nb MMAs per stage
//               (A = W from TMEM, B = X from shared memory) and commits the
//               X and W slots.
//   warp 8      also allocates / frees TMEM
//   warps 12-19 epilogue: per chunk tcgen05.ld of the finished accumulator
//               (lane quadrant w % 4, column half), add, release.
// TMEM: accumulators [0, fpass) and [208, 208 + fpass), W slots 416 + 32 s
// (s < 3; per slot kb x {hi, lo} x 8 columns of fp16 pairs).
// IQ16 layout (demod_fused_kernel<., true>): [a][e][TP / 4 row chunks][plane
// hi|lo][frame][4 rows x (re, im)] fp16, the stored rows iq_row0 .. iq_row0
// + TP - 1 (TP = iq_rows rounded to 4, pad rows zero).  A window of chunks is
// one contiguous run of both planes, and a chunk of one plane in shared
// memory the canonical no-swizzle K-major operand (8-frame x 16 B core
// matrices, SBO 128 B; LBO = two chunks, the other plane's in between).
// Measurements and the design's history: profiles/r02_das_tc_C.md.
#include <cuda_fp16.h>

namespace fqfg {

// Protocol / bounds checks, compiled in only for the checked build (`make
// check` -> libfqfgpu_check.so; scripts/gpu/checked_das.sh): compute-sanitizer
// is not available on this GPU pool.
#ifdef FQFG_TC_CHECK
#define TC_CHECK(cond)                                                                      \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("das_tc check failed: %s (block %d thread %d)\n", #cond, blockIdx.x, threadIdx.x); \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define TC_CHECK(cond) \
  do {                 \
  } while (0)
#endif

constexpr int kTcV = 64;
constexpr int kTcNS = 3;   // W slots in TMEM
constexpr int kTcMaxNX = 6;  // X slots in shared memory (as many as fit)
constexpr int kTcChunk = 16;
constexpr int kTcMaxTB = 4;  // table buffers (blocks computed ahead of the emitter): 4, 3, or 2 if
                             // the tables of many angles leave too little shared memory
constexpr int kTcEB = 3;  // elements per table block: 3 x 64 voxels = the 192 table threads
constexpr int kTcMaxA = 16;
constexpr int kTcXSlot = 2 * 4 * 208 * 16;  // X slot: {hi, lo} x 4 row chunks x fpass x 16 B
constexpr int kTcWarps = 20;
constexpr int kTcAcc1 = 208;   // second accumulator's first TMEM column
constexpr int kTcWCol = 416;   // first W slot column
constexpr int kTcMaxFpass = 208;

struct TcHdr {
  int done, nb, t_base, tab;  // tab: first float4 of the stage's 64 table entries
  int lim;                    // taps with r0 >= lim belong to the next part
  int release;                // table buffer the W writers release, -1 none
  int pad[2];
};

struct TcSmem {
  int x_off, tab_off, vox_off, ttx_off, tb_off, win_off, lst_off, hdr_off, bar_off, misc_off,
      total;
  __host__ __device__ TcSmem(int A, int NX, int TB) {
    auto up = [](int v) { return (v + 127) & ~127; };  // 128-byte aligned regions
    x_off = 0;
    tab_off = x_off + NX * kTcXSlot;
    vox_off = up(tab_off + TB * kTcEB * A * kTcV * 16);
    ttx_off = up(vox_off + kTcV * 24);
    tb_off = up(ttx_off + A * kTcV * 8);
    win_off = up(tb_off + A * 16);
    lst_off = up(win_off + TB * kTcEB * A * 2 * 8);
    hdr_off = up(lst_off + TB * kTcEB * A * 16);
    bar_off = up(hdr_off + kTcMaxNX * (int)sizeof(TcHdr));
    misc_off = up(bar_off + (3 * kTcMaxNX + 2 * kTcNS + 2 * kTcMaxTB + 4) * 8);
    total = misc_off + 128;
  }
};
inline size_t das_tc_smem(int A, int NX, int TB) { return (size_t)TcSmem(A, NX, TB).total + 1024; }
// Table buffers and X slots that fit (4 x 4 at 9 angles, 2 x 4 at 15):
// packed as TB << 8 | NX (DasLaunch::rcap), 0 if even 2 x 3 do not fit.
inline int das_tc_slots(int A, int max_smem) {
  for (int tb = kTcMaxTB; tb >= 3; --tb)
    for (int nx = kTcMaxNX; nx >= 4; --nx)  // four or three table buffers with >= 4 X slots
      if (das_tc_smem(A, nx, tb) <= (size_t)max_smem) return tb << 8 | nx;
  for (int nx = kTcMaxNX; nx >= 3; --nx)  // else two
    if (das_tc_smem(A, nx, 2) <= (size_t)max_smem) return 2 << 8 | nx;
  return 0;
}

FQFG_DEVICE uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}

// D (+)= A B with A (M = 128 x K = 16 fp16) in TMEM and B from shared memory.
FQFG_DEVICE void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                           uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

FQFG_DEVICE void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

FQFG_DEVICE void mbar_arrive_n(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(n)
               : "memory");
}

FQFG_DEVICE void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}

// One thread of the (converged) warp: elect.sync, which ptxas knows to be a
// single lane, so the guarded tcgen05 operands need no per-lane loop.
FQFG_DEVICE bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(e));
  return e != 0;
}

FQFG_DEVICE uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// Warp-group register split (setmaxnreg): emitter/table and MMA/table 80,
// W writers 64, epilogue 128 (104 fp32 accumulators per thread).
constexpr int kTcRegProd = 80, kTcRegW = 64, kTcRegEpi = 128;

__global__ void __launch_bounds__(kTcWarps * 32, 1)
    das_tc_kernel(const DasParams p, const DasLaunch L, const __half* __restrict__ iq16,
                  const float* __restrict__ d_scale, float2* __restrict__ x,
                  unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base =
      smem_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  const int NX = L.rcap & 0xff, TB = L.rcap >> 8;  // X slots, table buffers
  const TcSmem S(p.A, NX, TB);
  unsigned char* xs = base + S.x_off;
  float4* tab = reinterpret_cast<float4*>(base + S.tab_off);  // [TB][EB][A][64]
  double* vox = reinterpret_cast<double*>(base + S.vox_off);  // [64][3]
  double* ttxA = reinterpret_cast<double*>(base + S.ttx_off);  // [A][64]
  double* tbound = reinterpret_cast<double*>(base + S.tb_off);  // [A][2]
  int2* win = reinterpret_cast<int2*>(base + S.win_off);  // [TB][EB][A][2] (first, last) tap row
  // [TB][EB A] windows of a table block with taps: (chunk of its first row in
  // plane 0, sample of its first row, table index, rows); count in lcnt[TB]
  int4* lst = reinterpret_cast<int4*>(base + S.lst_off);
  TcHdr* hdr = reinterpret_cast<TcHdr*>(base + S.hdr_off);     // [NX]
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + S.bar_off);
  uint64_t* hfull = bars;                  // [NX] header published (count 1)
  uint64_t* xfull = hfull + kTcMaxNX;      // [NX] X landed (count 1 + tx)
  uint64_t* xempty = xfull + kTcMaxNX;     // [NX] MMAs done with the X slot (count 1)
  uint64_t* wfull = xempty + kTcMaxNX;     // [NS] W in TMEM (count 4)
  uint64_t* wempty = wfull + kTcNS;        // [NS] MMAs done with the W slot (count 1)
  uint64_t* tready = wempty + kTcNS;       // [TB] table block ready (count 1)
  uint64_t* tempty = tready + kTcMaxTB;    // [TB] table block released (count 4)
  uint64_t* accfull = tempty + kTcMaxTB;   // [2] (count 2)
  uint64_t* accempty = accfull + 2;        // [2] (count 8)
  int* misc = reinterpret_cast<int*>(base + S.misc_off);
  // misc: [0] tmem, [1..2] nst, [3..4] fin
  int* lcnt = misc + 5;  // [TB] stages in the list of each table buffer

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fpass = p.fpass;
  int tile = blockIdx.x;
  const int tx = tile % L.tiles_x;
  tile /= L.tiles_x;
  const int ty = tile % L.tiles_y;
  const int ntz = (L.kend - L.kbeg + L.TZ - 1) / L.TZ;
  const int tz = ntz - 1 - tile / L.tiles_y;  // deep planes first (das2)
  const int i0 = tx * L.TX, j0 = ty * L.TY, k0 = L.kbeg + tz * L.TZ;

  // X slots start zeroed: a K block's unloaded half-chunk holds finite data
  // (W is zero there)
  for (int i = tid; i < NX * kTcXSlot / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(xs)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int l = tid; l < kTcV; l += blockDim.x) {
    const int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
    const int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    const bool ok = i < p.nx && j < p.ny && k < L.kend;
    vox[3 * l] = ok ? grid_coord(p.ox, i, p.sx) : __longlong_as_double(0x7ff8000000000000ll);
    vox[3 * l + 1] = grid_coord(p.oy, j, p.sy);
    vox[3 * l + 2] = grid_coord(p.oz, k, p.sz);
  }
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(&hfull[s], 1);
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < kTcNS; ++s) {
      mbar_init(&wfull[s], 4);
      mbar_init(&wempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 2);
      mbar_init(&accempty[b], 8);
    }
    for (int b = 0; b < TB; ++b) {
      mbar_init(&tready[b], 1);
      mbar_init(&tempty[b], 4);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(misc)));
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
  // Tile box and its transmit-delay range per angle (das2).
  const int i1 = min(i0 + L.TX, p.nx) - 1, j1 = min(j0 + L.TY, p.ny) - 1,
            k1 = min(k0 + L.TZ, L.kend) - 1;
  const double bx0 = grid_coord(p.ox, i0, p.sx), bx1 = grid_coord(p.ox, i1, p.sx);
  const double by0 = grid_coord(p.oy, j0, p.sy), by1 = grid_coord(p.oy, j1, p.sy);
  const double bz0 = grid_coord(p.oz, k0, p.sz), bz1 = grid_coord(p.oz, k1, p.sz);
  for (int a = tid; a < p.A; a += blockDim.x) {
    const AngleConst ac = p.ang[a];
    tbound[2 * a] = (fmin(bx0 * ac.sina, bx1 * ac.sina) + bz0 * ac.cosa - ac.ref) / p.c;
    tbound[2 * a + 1] = (fmax(bx0 * ac.sina, bx1 * ac.sina) + bz1 * ac.cosa - ac.ref) / p.c;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  const int nblk = (p.E + kTcEB - 1) / kTcEB;
  const int NRB = ((p.iq_rows + 3) & ~3) >> 2;  // stored row chunks per (plane, a, e)
  const int AV = p.A * kTcV;
  const int span = 12;  // part stride (rows): parts overlap by 4, a tap pair never straddles

  // ============================ table ============================
  // (warps 2-3 and 8-11: NT threads, tt = index in the group)
  constexpr int NT = 192;
  auto table_role = [&](const int tt) {
    // thread tt owns (element tt / 64 of the block, voxel tt % 64): its
    // receive delay / aperture test, then its entries for every angle (A
    // independent chains); no barrier until the block is complete
    unsigned long long n_oow = 0, n_taps = 0;
    const int el = tt / kTcV, v = tt % kTcV, tw = tt >> 5;
    const double px = vox[3 * v], py = vox[3 * v + 1], pz = vox[3 * v + 2];
    for (int blk = 0; blk < nblk; ++blk) {
      const int buf = blk % TB;
      if (blk >= TB) mbar_wait_sleep(&tempty[buf], ((blk / TB) - 1) & 1, 256);
      const int e0 = blk * kTcEB, e = e0 + el;
      double r = -1.0;
      if (e < p.E && px == px) {
        const double ex = __ldg(p.elem + 3 * e), ey = __ldg(p.elem + 3 * e + 1),
                     ez = __ldg(p.elem + 3 * e + 2);
        if (!(p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum)))
          r = rx_delay(px, py, pz, ex, ey, ez, p.c);
      }
      float4* tb = tab + (size_t)buf * kTcEB * AV + el * AV + v;
      // (every lane runs the angle loop: the row bounds are warp reductions;
      // not unrolled: the table warps share issue slots with the serial
      // roles, unroll 3 / 4 / 5 measured 2 / 7 / 7 % slower at config B)
#pragma unroll 1
      for (int a = 0; a < p.A; ++a) {
        float4 ent = make_float4(__int_as_float(kInactive), 0.f, 0.f, 0.f);
        int first = 0x7fffffff, last = (int)0x80000000;
        if (r >= 0.0) {
          const AngleConst ac = p.ang[a];
          const double tau = xadd(ttxA[a * kTcV + v], r);
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
            first = s0;
            last = frac > 0.f ? s0 + 1 : s0;
          }
        }
        tb[a * kTcV] = ent;
        // exact tap rows of the (element, angle) over this warp's 32 voxels
        first = __reduce_min_sync(0xffffffffu, first);
        last = __reduce_max_sync(0xffffffffu, last);
        if (lane == 0) win[((buf * kTcEB + el) * p.A + a) * 2 + (tw & 1)] = make_int2(first, last);
      }
      named_sync(2, NT);
      if (tw == 0) {
        // window list of the block, in (element, angle) order: rows from the
        // exact tap rows of both table warps, starting on a stored row that
        // is a multiple of 4 (chunk)
        const int cap = kTcEB * p.A;
        int4* L4 = lst + (size_t)buf * cap;
        int base_k = 0;
        for (int i0 = 0; i0 < cap; i0 += 32) {
          const int i = i0 + lane;
          int4 ent = make_int4(0, 0, 0, 0);
          bool has = false;
          if (i < cap) {
            const int wel = i / p.A, a = i % p.A;
            const int2 w0 = win[((buf * kTcEB + wel) * p.A + a) * 2];
            const int2 w1 = win[((buf * kTcEB + wel) * p.A + a) * 2 + 1];
            const int first = min(w0.x, w1.x), last = max(w0.y, w1.y);
            if (first <= last) {
              const int lo_sr = (first + 1 - p.iq_row0) & ~3;
              TC_CHECK(first + 1 - p.iq_row0 >= 0 && (lo_sr >> 2) < NRB && last >= first);
              const int lo = lo_sr - 1 + p.iq_row0;  // sample of the first window row
              ent = make_int4((a * p.E + e0 + wel) * NRB + (lo_sr >> 2), lo,
                              ((buf * kTcEB + wel) * p.A + a) * kTcV, last - lo + 1);
              has = true;
            }
          }
          const unsigned bal = __ballot_sync(0xffffffffu, has);
          if (has) L4[base_k + __popc(bal & ((1u << lane) - 1u))] = ent;
          base_k += __popc(bal);
        }
        if (lane == 0) lcnt[buf] = base_k;
        __syncwarp();
        if (lane == 0) mbar_arrive(&tready[buf]);
      }
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
  };

  if (warp < 4 && warp != 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kTcRegProd));
    if (warp == 0) {
      // ========================== stage emitter ==========================
      int pend = -1;
      // nch: 4-row chunks to load (nb = ceil(nch / 2) K blocks)
      // (the whole warp walks the stages, warp-uniform values; one elected
      // thread publishes the header and issues the copies)
      int eslot = 0;
      unsigned eph = 0;
      unsigned long long nkb = 0;  // K blocks emitted (roofline instrumentation)
      const unsigned hdr_s = (unsigned)__cvta_generic_to_shared(hdr);
      const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bars);  // hfull; xfull at + kTcMaxNX
      const unsigned xs_s = (unsigned)__cvta_generic_to_shared(xs);
      auto emit = [&](int nch, int t_base, int tabi, int lim, int c2) {
        const int nb = nch < 0 ? -1 : (nch + 1) / 2;
        if (nb > 0) nkb += (unsigned long long)nb;
        const int slot = eslot;
        mbar_wait(&xempty[slot], eph ^ 1);
        // one elected lane, predicated (no divergent branch): header,
        // hfull, then the window's chunks (both planes of a chunk are
        // adjacent and the chunks of an (a, e) consecutive: one bulk copy of
        // nch x 2 x fpass x 16 B from chunk c2; the buffer is padded past the
        // last element, rows past the window carry zero weights) or a plain
        // xfull arrive
        const unsigned bytes = nch > 0 ? (unsigned)(nch * 2 * fpass * 16) : 0u;
        // the copy stays inside the IQ16 buffer (+ its 4-chunk pad), the slot
        // and the table block
        TC_CHECK(nch <= 0 || (nch <= 4 && c2 >= 0 &&
                              (long long)c2 + nch <= (long long)p.A * p.E * NRB + 4 &&
                              tabi >= 0 && tabi + kTcV <= TB * kTcEB * AV && lim >= 1 && lim <= 16));
        const unsigned long long src0 =
            (unsigned long long)(iq16 + (size_t)(unsigned)c2 * (unsigned)(2 * fpass * 8));
        const unsigned dst0 = xs_s + (unsigned)(slot * kTcXSlot);
        asm volatile(
            "{\n.reg .pred P, Q, PQ, PN;\n"
            "elect.sync _|P, 0xffffffff;\n"
            "setp.gt.s32 Q, %2, 0;\n"
            "and.pred PQ, P, Q;\n"
            "and.pred PN, P, !Q;\n"
            "@P st.shared.v4.b32 [%0], {%3, %4, %5, %6};\n"
            "@P st.shared.v4.b32 [%0 + 16], {%7, %8, 0, 0};\n"
            "@P mbarrier.arrive.shared::cta.b64 _, [%1];\n"
            "@PQ mbarrier.arrive.expect_tx.shared::cta.b64 _, [%9], %10;\n"
            "@PQ cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%11], [%12], %10, [%9];\n"
            "@PN mbarrier.arrive.shared::cta.b64 _, [%9];\n"
            "}\n" ::"r"(hdr_s + (unsigned)(slot * (int)sizeof(TcHdr))),
            "r"(bar_s + (unsigned)(slot * 8)), "r"(nb), "r"(nb < 0 ? 1 : 0), "r"(nb < 0 ? 0 : nb),
            "r"(t_base), "r"(tabi), "r"(lim), "r"(pend), "r"(bar_s + (unsigned)((kTcMaxNX + slot) * 8)),
            "r"(bytes), "r"(dst0), "l"(src0)
            : "memory");
        pend = -1;
        if (++eslot == NX) eslot = 0, eph ^= 1;
      };
      for (int blk = 0; blk < nblk; ++blk) {
        const int buf = blk % TB;
        mbar_wait(&tready[buf], (blk / TB) & 1);
        const int cnt = lcnt[buf];
        const int4* L4 = lst + (size_t)buf * kTcEB * p.A;
        const bool any = cnt > 0;
        for (int k = 0; k < cnt; ++k) {
          // parts of <= 16 rows every 12 (3 chunks): a tap pair never
          // straddles two parts; taps with r0 >= lim belong to the next
          const int4 wn = L4[k];
          const int n = wn.w;
          const int nparts = n <= 16 ? 1 : 1 + (n - 16 + span - 1) / span;
          for (int part = 0; part < nparts; ++part) {
            const int rows = min(16, n - part * span);
            emit((rows + 3) / 4, wn.y + part * span, wn.z, part + 1 == nparts ? 16 : span,
                 wn.x + 3 * part);
          }
        }
        if (any) {
          pend = buf;  // released by the W writers with the next stage they read
        } else {
          // nobody reads this table; a release still pending from an earlier
          // block goes out on a no-op stage (the table warps may need that
          // buffer before another stage comes)
          if (pend >= 0) emit(0, 0, 0, 0, 0);
          if (elect_one()) mbar_arrive_n(&tempty[buf], 4);
          __syncwarp();
        }
      }
      emit(-1, 0, 0, 0, 0);  // termination (carries the last release)
      if (L.kblocks && elect_one()) atomicAdd(L.kblocks, nkb);
      __syncwarp();
    } else {
      table_role(tid - 64);
    }
  } else if (warp >= 4 && warp < 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kTcRegW));
    // ============================ W writers ============================
    const int q = warp - 4;
    const int m = 32 * q + lane, v = m & 63, c = m >> 6;
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    int xsl = 0, slot = 0;
    unsigned xph = 0, wph = 0;
    for (;;) {
      mbar_wait(&hfull[xsl], xph);
      const TcHdr h = hdr[xsl];
      TC_CHECK(h.done || (h.nb >= 0 && h.nb <= 2 && h.release >= -1 && h.release < TB));
      if (h.done) {
        if (h.release >= 0 && lane == 0) mbar_arrive(&tempty[h.release]);
        break;
      }
      // the W slot is free once the MMAs of stage - NS are complete
      mbar_wait(&wempty[slot], wph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (h.nb > 0) {
        const float4 ent = tab[h.tab + v];
        const int s0 = __float_as_int(ent.x);
        const int r0 = s0 == kInactive ? -100 : s0 - h.t_base;
        const bool act = s0 != kInactive && r0 >= 0 && r0 < h.lim;
        const float fr = ent.y, cr = ent.z, ci = ent.w, w0 = 1.0f - fr;
        // (re row) Wr x_re - Wi x_im ; (im row) Wi x_re + Wr x_im, per tap
        const float q0 = c ? ci * w0 : cr * w0, q1 = c ? cr * w0 : -(ci * w0);
        const float q2 = c ? ci * fr : cr * fr, q3 = c ? cr * fr : -(ci * fr);
        const __half2 h01 = __floats2half2_rn(q0, q1), h23 = __floats2half2_rn(q2, q3);
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        const uint32_t H0 = act ? h2u(h01) : 0u, H1 = act ? h2u(h23) : 0u;
        const uint32_t L0 = act ? h2u(__floats2half2_rn(q0 - f01.x, q1 - f01.y)) : 0u;
        const uint32_t L1 = act ? h2u(__floats2half2_rn(q2 - f23.x, q3 - f23.y)) : 0u;
        // words of K block kb (hi columns 0-7, lo 8-15): row r = 8 kb + col
        auto block_words = [&](int kb, uint32_t (&w)[16]) {
          // word j (hi) / 8 + j (lo) of the K block: tap 0 if j == r0 - 8 kb,
          // tap 1 if j == r0 - 8 kb + 1, else 0 -- nine compares and two
          // selects per word (PTX: C ternaries here would become branches)
          asm("{\n.reg .pred e0, e1, e2, e3, e4, e5, e6, e7, e8;\n"
              "setp.eq.s32 e0, %20, -1;\n"
              "setp.eq.s32 e1, %20, 0;\n"
              "setp.eq.s32 e2, %20, 1;\n"
              "setp.eq.s32 e3, %20, 2;\n"
              "setp.eq.s32 e4, %20, 3;\n"
              "setp.eq.s32 e5, %20, 4;\n"
              "setp.eq.s32 e6, %20, 5;\n"
              "setp.eq.s32 e7, %20, 6;\n"
              "setp.eq.s32 e8, %20, 7;\n"
              "selp.b32 %0, %17, 0, e0;\n"
              "selp.b32 %0, %16, %0, e1;\n"
              "selp.b32 %8, %19, 0, e0;\n"
              "selp.b32 %8, %18, %8, e1;\n"
              "selp.b32 %1, %17, 0, e1;\n"
              "selp.b32 %1, %16, %1, e2;\n"
              "selp.b32 %9, %19, 0, e1;\n"
              "selp.b32 %9, %18, %9, e2;\n"
              "selp.b32 %2, %17, 0, e2;\n"
              "selp.b32 %2, %16, %2, e3;\n"
              "selp.b32 %10, %19, 0, e2;\n"
              "selp.b32 %10, %18, %10, e3;\n"
              "selp.b32 %3, %17, 0, e3;\n"
              "selp.b32 %3, %16, %3, e4;\n"
              "selp.b32 %11, %19, 0, e3;\n"
              "selp.b32 %11, %18, %11, e4;\n"
              "selp.b32 %4, %17, 0, e4;\n"
              "selp.b32 %4, %16, %4, e5;\n"
              "selp.b32 %12, %19, 0, e4;\n"
              "selp.b32 %12, %18, %12, e5;\n"
              "selp.b32 %5, %17, 0, e5;\n"
              "selp.b32 %5, %16, %5, e6;\n"
              "selp.b32 %13, %19, 0, e5;\n"
              "selp.b32 %13, %18, %13, e6;\n"
              "selp.b32 %6, %17, 0, e6;\n"
              "selp.b32 %6, %16, %6, e7;\n"
              "selp.b32 %14, %19, 0, e6;\n"
              "selp.b32 %14, %18, %14, e7;\n"
              "selp.b32 %7, %17, 0, e7;\n"
              "selp.b32 %7, %16, %7, e8;\n"
              "selp.b32 %15, %19, 0, e7;\n"
              "selp.b32 %15, %18, %15, e8;\n"
              "}\n"
              : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]),
                "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
              : "r"(H0), "r"(H1), "r"(L0), "r"(L1), "r"(r0 - 8 * kb));
        };
        const uint32_t ta = trow + (uint32_t)(kTcWCol + 32 * slot);
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          if (kb < h.nb) {
            uint32_t w[16];
            block_words(kb, w);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                "%12,%13,%14,%15,%16};" ::"r"(ta + 16 * kb),
                "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                "r"(w[14]), "r"(w[15])
                : "memory");
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&wfull[slot]);
        if (h.release >= 0) mbar_arrive(&tempty[h.release]);
      }
      if (++xsl == NX) xsl = 0, xph ^= 1;
      if (++slot == kTcNS) slot = 0, wph ^= 1;
    }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kTcRegProd));
    if (warp >= 8) {
      table_role(64 + tid - 8 * 32);
    } else {
      // =============================== MMA ===============================
      // The whole warp walks the stages (warp-uniform slot indices, phases and
      // descriptors, so the operands stay in uniform registers); one elected
      // thread issues the MMAs and commits.
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      // idesc: D f32 (1 << 4), A f16, B f16, K-major, N = fpass, M = 128
      const uint32_t idesc = (1u << 4) | ((uint32_t)(fpass >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t chunk_b = (uint32_t)fpass * 16;
      // X slot: chunk j of plane hi at 2 j chunk_b, of plane lo at (2 j + 1)
      // chunk_b: a K block's two chunks are LBO = 2 chunk_b apart
      const uint64_t xdesc0 = umma_desc_kmajor((uint32_t)__cvta_generic_to_shared(xs), 2 * chunk_b);
      const uint64_t dk1 = (uint64_t)((4 * chunk_b) >> 4);  // K block 1 (chunks 2, 3)
      const uint64_t dlo = (uint64_t)(chunk_b >> 4);        // lo plane
      const uint64_t dslot = (uint64_t)(kTcXSlot >> 4);
      int chunk = 0, in_chunk = 0;
      int xsl = 0, wsl = 0;
      unsigned xph = 0, wph = 0;
      for (;;) {
        mbar_wait(&xfull[xsl], xph);
        const int b = chunk & 1;
        const int2 hd = *reinterpret_cast<const int2*>(&hdr[xsl]);  // (done, nb)
        const int done = __shfl_sync(0xffffffffu, hd.x, 0), nb = __shfl_sync(0xffffffffu, hd.y, 0);
        TC_CHECK(done || (nb >= 0 && nb <= 2));
        if (done) {
          // (the epilogue must have taken chunk - 2 out of buffer b first)
          if (in_chunk == 0 && chunk >= 2) mbar_wait(&accempty[b], ((chunk >> 1) - 1) & 1);
          if (elect_one()) {
            misc[1 + b] = in_chunk;
            misc[3 + b] = 1;
            tc_commit(&accfull[b]);
            mbar_arrive(&accfull[b]);
          }
          __syncwarp();
          break;
        }
        mbar_wait(&wfull[wsl], wph);
        if (in_chunk == 0 && chunk >= 2) mbar_wait(&accempty[b], ((chunk >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (elect_one()) {
          if (nb > 0) {
            const uint32_t d = tm + (uint32_t)(kTcAcc1 * b);
            const uint32_t wa = tm + (uint32_t)(kTcWCol + 32 * wsl);
            const uint64_t xd = xdesc0 + dslot * (uint64_t)xsl;
            tc_mma_ts(d, wa, xd, idesc, in_chunk > 0 ? 1u : 0u);
            tc_mma_ts(d, wa, xd + dlo, idesc, 1u);
            tc_mma_ts(d, wa + 8, xd, idesc, 1u);
            if (nb > 1) {
              tc_mma_ts(d, wa + 16, xd + dk1, idesc, 1u);
              tc_mma_ts(d, wa + 16, xd + dk1 + dlo, idesc, 1u);
              tc_mma_ts(d, wa + 24, xd + dk1, idesc, 1u);
            }
            tc_commit(&xempty[xsl]);
            tc_commit(&wempty[wsl]);
          } else {
            mbar_arrive(&xempty[xsl]);
            mbar_arrive(&wempty[wsl]);
          }
        }
        __syncwarp();
        if (++xsl == NX) xsl = 0, xph ^= 1;
        if (++wsl == kTcNS) wsl = 0, wph ^= 1;
        if (nb > 0 && ++in_chunk == kTcChunk) {
          if (elect_one()) {
            misc[1 + b] = in_chunk;
            misc[3 + b] = 0;
            tc_commit(&accfull[b]);
            mbar_arrive(&accfull[b]);
          }
          __syncwarp();
          in_chunk = 0;
          ++chunk;
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kTcRegEpi));
    // ============================ epilogue ============================
    const int q = warp & 3, half = (warp - 12) >> 2;
    const int m = 32 * q + lane;
    const int ncol = fpass / 2;  // columns of this thread (<= 104)
    float acc[104];
#pragma unroll
    for (int j = 0; j < 104; ++j) acc[j] = 0.f;
    for (int chunk = 0;; ++chunk) {
      const int b = chunk & 1;
      // (idle between drains: sleep between probes instead of spinning)
      mbar_wait_sleep(&accfull[b], (chunk >> 1) & 1, 512);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int nst = misc[1 + b], fin = misc[3 + b];
      if (nst > 0) {
        const uint32_t taddr =
            tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(kTcAcc1 * b + half * ncol);
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
    // x[f][voxel - x_v0] (re for m < 64, im for m >= 64) = acc / (A S_f)
    const int v = m & 63, c = m >> 6;
    const int lx = v % L.TX, ly = (v / L.TX) % L.TY, lz = v / (L.TX * L.TY);
    const int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    if (i < p.nx && j < p.ny && k < L.kend) {
      const float invA = (float)(1.0 / p.A);
      const size_t flat =
          (size_t)((long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * k) - L.x_v0);
      float* xo = reinterpret_cast<float*>(x);
#pragma unroll
      for (int jj = 0; jj < 104; ++jj) {
        const int fl = half * ncol + jj;
        const int f = L.pass * fpass + fl;
        if (jj < ncol && f < p.F)
          xo[2 * ((size_t)f * (size_t)L.x_n + flat) + c] = acc[jj] * invA / __ldg(d_scale + fl);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Per-frame max |RF| over the source window of frames [f_lo, f_lo + nv) of
// the pass (all angles, rows [t0, t0 + rows), elements) -> mx[frame of the
// pass] (float bits, atomicMax; mx zeroed by the caller).  grid (blocks per
// angle window, nv, A): each (frame, angle) window is one contiguous run of
// rows x E floats, read as float4 when it is 16-byte aligned.
__global__ void __launch_bounds__(256) rf_frame_absmax_kernel(const RfSrc src, int A, int E,
                                                              int f_lo, unsigned* __restrict__ mx) {
  const int fr = blockIdx.y, a = blockIdx.z;
  const size_t n = (size_t)src.rows * E;
  const float* rf = src.rf + (long long)(f_lo + fr - src.f_base) * src.fst + (long long)a * src.sst;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  float m = 0.f;
  if ((reinterpret_cast<uintptr_t>(rf) & 15) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(rf);
    const size_t n4 = n / 4;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldg(r4 + i);
      const float b = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
      m = b == b ? fmaxf(m, b) : m;  // (NaN-free max, as the scalar path)
    }
    for (size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const float v = fabsf(rf[i]);
      m = v == v ? fmaxf(m, v) : m;
    }
  } else {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const float v = fabsf(rf[i]);
      m = v == v ? fmaxf(m, v) : m;
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx + f_lo + fr, __float_as_uint(m));
}

// S_f = 2^floor(log2(6e4 / (2 sum|h| max|RF_f|))) for frames [f_lo, f_lo + n)
// (1 for empty / padding frames): |IQ S_f| <= 6e4, inside the fp16 range.
__global__ void tc_scale_kernel(const unsigned* __restrict__ mx, float hsum, int f_lo, int n,
                                float* __restrict__ s) {
  const int f = f_lo + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (f >= f_lo + n) return;
  const float bound = 2.f * hsum * __uint_as_float(mx[f]);
  float sc = 1.f;
  if (bound > 0.f && isfinite(bound)) {
    const float e = floorf(log2f(6.0e4f / bound));
    sc = exp2f(fminf(fmaxf(e, -100.f), 100.f));
  }
  s[f] = sc;
}

}  // namespace fqfg
