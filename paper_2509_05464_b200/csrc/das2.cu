// das2.cu -- warp-specialised, double-buffered DAS (the production kernel).
//
// Same semantics and the same reference-exact FP64 delay geometry as
// das_kernel (das.cu; das.cpp:126-222, 309-328), restructured so that the
// three costs of a stage overlap instead of serialising behind
// __syncthreads():
//
//   producer warpgroup (4 warps)   per stage s = (element block eb, angle a):
//     wait empty[s%NS]; FP64 tap index / weight / carrier rotation for every
//     (voxel, element) -> table slot; per-element window [min s0, max s0 + 1];
//     one elected thread packs the windows into the slot's row buffer and
//     issues 1-D TMA bulk copies (cp.async.bulk) completing on full[s%NS].
//   consumer warps (NCW)           per stage: wait full[s%NS]; gather the two
//     taps of every (voxel, element, frame) from shared memory (lanes = 16
//     frames x 2 voxels), interpolate, rotate, accumulate in registers;
//     arrive empty[s%NS].
//
// NS = 2 slots, so the TMA copy and the FP64 table of stage s+1 run while the
// consumers gather stage s.  Elements whose window does not fit the slot are
// gathered straight from global memory (same arithmetic).
#include "common.cuh"

namespace fqfg {

FQFG_DEVICE void mbar_arrive(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// v = *addr (shared memory) when p, else v unchanged -- a predicated load, so
// the row-cache refresh of mode 2 needs no branch.
FQFG_DEVICE void lds_if(unsigned p, float2& v, unsigned addr) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q ld.shared.v2.f32 {%0, %1}, [%3];\n\t}"
      : "+f"(v.x), "+f"(v.y)
      : "r"(p), "r"(addr));
}

FQFG_DEVICE void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- TMEM (tensor memory) accumulators for mode 4 ----
// tcgen05.ld / tcgen05.st of N consecutive 32-bit columns of this warp's lane
// quadrant (32x32b shape: thread i <-> TMEM lane 32 (warp % 4) + i).
#define FQFG_R16(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), \
    "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),   \
    "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
#define FQFG_W16(r) "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), \
    "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),             \
    "r"(r[14]), "r"(r[15])
template <int N>
FQFG_DEVICE void tm_ld(uint32_t a, uint32_t* r) {
  if constexpr (N >= 16) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                 "%12,%13,%14,%15}, [%16];"
                 : FQFG_R16(r)
                 : "r"(a));
    tm_ld<N - 16>(a + 16, r + 16);
  } else if constexpr (N >= 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
    tm_ld<N - 8>(a + 8, r + 8);
  } else if constexpr (N >= 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
    tm_ld<N - 4>(a + 4, r + 4);
  } else if constexpr (N >= 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(a));
    tm_ld<N - 2>(a + 2, r + 2);
  } else if constexpr (N == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(a));
  }
}
template <int N>
FQFG_DEVICE void tm_st(uint32_t a, const uint32_t* r) {
  if constexpr (N >= 16) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
                 "%11,%12,%13,%14,%15,%16};" ::"r"(a),
                 FQFG_W16(r)
                 : "memory");
    tm_st<N - 16>(a + 16, r + 16);
  } else if constexpr (N >= 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                 "r"(r[7])
                 : "memory");
    tm_st<N - 8>(a + 8, r + 8);
  } else if constexpr (N >= 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
    tm_st<N - 4>(a + 4, r + 4);
  } else if constexpr (N >= 2) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(a), "r"(r[0]),
                 "r"(r[1])
                 : "memory");
    tm_st<N - 2>(a + 2, r + 2);
  } else if constexpr (N == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "r"(r[0])
                 : "memory");
  }
}
// Packed FP32 pairs (FFMA2 on sm_100): a float2 held in one 64-bit register.
FQFG_DEVICE unsigned long long f2pk(uint32_t lo, uint32_t hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
FQFG_DEVICE void f2upk(unsigned long long r, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(r));
}
FQFG_DEVICE unsigned long long f2bc(float a) { return f2pk(__float_as_uint(a), __float_as_uint(a)); }
FQFG_DEVICE unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                     unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

FQFG_DEVICE void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
FQFG_DEVICE void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }


// Register split between the producer and consumer warpgroups (setmaxnreg):
// the launch gives every thread R0 registers; producers drop to kProdRegs and
// consumers take the rest.
constexpr int das2_launch_regs(int warps) {
  return ((65536 / (32 * warps)) / 8 * 8) > 248 ? 248 : (65536 / (32 * warps)) / 8 * 8;
}
constexpr int das2_prod_regs(int pw, int ncw) { return pw == 4 && ncw <= 8 ? 80 : 64; }
constexpr int das2_cons_regs(int ncw, int pw) {
  return (((ncw + pw) * das2_launch_regs(ncw + pw) - pw * das2_prod_regs(pw, ncw)) / ncw / 8 * 8) >
                 248
             ? 248
             : ((ncw + pw) * das2_launch_regs(ncw + pw) - pw * das2_prod_regs(pw, ncw)) / ncw / 8 *
                   8;
}

// Tile-local voxel coordinates of table index l.  Mode 0: x fastest.
// Mode 3: y fastest, so each y-column of VPW voxels is a contiguous range of
// table entries.
template <int MODE>
FQFG_DEVICE void tile_local(int l, const DasLaunch& L, int& lx, int& ly, int& lz) {
  if (MODE >= 3) {
    ly = l % L.TY;
    lx = (l / L.TY) % L.TX;
    lz = l / (L.TX * L.TY);
  } else {
    lx = l % L.TX;
    ly = (l / L.TX) % L.TY;
    lz = l / (L.TX * L.TY);
  }
}

struct SlotHdr {
  int done, eb, a, pad;
  int wbase[8];  // >= 0 row in slot buffer, -1 gather from global, -2 element unused
  int wmin[8];
  int wmax[8];
};

// MODE 0: lanes = 16 frames x 2 voxels (half-warps), fpass = 16 J.
// MODE 3: lanes = 16 frames x 2 half-warps; each half-warp owns a y-column
//         of VPW voxels and keeps the two tap rows of the last voxel (x0 and
//         x1 - x0) in registers, reloading (both halves together, a
//         warp-uniform branch) only when a column's tap index changes
//         (|ds/dy| < 1 sample per voxel): ~0.7 instead of 2 rows per voxel.
//         Bitwise identical to mode 0; fewer shared-memory wavefronts but
//         more registers and branches (see profiles/r01_das2_C.md).
// (Lane mappings tried and dropped in round 1: 32 frame lanes with y-pair
//  sharing, and 32 frame lanes with a predicated row cache -- both slower.)
template <int J, int VPW, int NCW, int EB, int MODE, int NS, int PW>
__global__ void __launch_bounds__((NCW + PW) * 32, 1)
    das2_kernel(const DasParams p, const DasLaunch L, const float2* __restrict__ iq,
                float2* __restrict__ x, unsigned long long* __restrict__ counters) {
  // Mode 6: VPW voxels per consumer warp, NCW / 4 warps per TMEM lane quadrant.
  constexpr int V = MODE == 6 ? NCW / 4 * VPW : NCW * VPW * 2;
  static_assert(MODE != 3 || NCW % 4 == 0, "mode 3: tile = 8 x VPW x NCW/4 voxels");
  constexpr int NPT = PW * 32;
  static_assert(PW % 4 == 0 && NCW % 4 == 0, "setmaxnreg acts on whole warpgroups");
  static_assert(EB <= 8, "SlotHdr holds 8 elements");
  const int fpass = 16 * J;
  static_assert(MODE == 0 || MODE == 3 || MODE == 4 || MODE == 5 || MODE == 6,
                "lane mappings: 0 (voxel pairs), 3 (y-columns), 4 (y-columns, TMEM accumulators), "
                "5 (y-columns, TMEM, packed FP32)");
  static_assert(MODE != 4 || (NCW / 4) * VPW * 32 <= 512, "mode 4: TMEM holds 512 columns");
  static_assert(MODE != 5 || (NCW / 4) * VPW * 4 * J <= 512, "mode 5: TMEM holds 512 columns");
  static_assert(MODE != 6 || 16 * J <= 256, "mode 6: at most two 128-frame TMEM groups");
  const int rslot = L.rcap;  // rows per slot
  // Mode 6 stages each window as time-row pairs [pair][frame][2] plus a tail
  // pad (the second 128-frame group's tcgen05.cp reads 128 lanes).
  const int wstride = MODE == 6 ? rslot * fpass + 256 : rslot * fpass;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* win = reinterpret_cast<float2*>(smem_raw);  // [NS][wstride]
  unsigned char* sp = smem_raw + (size_t)NS * wstride * sizeof(float2);
  float4* tab = reinterpret_cast<float4*>(sp);         // [NS][EB][V]
  double* rc = reinterpret_cast<double*>(tab + NS * EB * V);  // [EB][V]
  double* vox = rc + EB * V;                           // [V][3]
  double* ttxA = vox + 3 * V;                          // [A][V] transmit delays
  double* tbound = ttxA + (size_t)p.A * V;             // [A][2] tile min/max ttx
  double* dbound = tbound + 2 * p.A;                   // [EB][2] |p-e|/c min/max
  SlotHdr* hdr = reinterpret_cast<SlotHdr*>(dbound + 2 * EB);  // [NS]
  uint64_t* full = reinterpret_cast<uint64_t*>(hdr + NS);
  uint64_t* empty = full + NS;
  int* flag = reinterpret_cast<int*>(empty + NS);
  int* exw = flag + 16;  // [NS][16]: exact-window tap-index min [0, 8) / max [8, 16) per element

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  int tile = blockIdx.x;
  const int tx = tile % L.tiles_x;
  tile /= L.tiles_x;
  const int ty = tile % L.tiles_y;
  // Deep planes first (L.debug bit 8 keeps the shallow-first order): deep tiles
  // see more elements inside the f-number cone and cost more, so the cheap
  // shallow tiles fill the last wave.
  const int ntz = (L.kend - L.kbeg + L.TZ - 1) / L.TZ;
  const int tz = (L.debug & 8) ? tile / L.tiles_y : ntz - 1 - tile / L.tiles_y;
  const int i0 = tx * L.TX, j0 = ty * L.TY, k0 = L.kbeg + tz * L.TZ;

  for (int l = tid; l < V; l += blockDim.x) {
    int lx, ly, lz;
    tile_local<MODE>(l, L, lx, ly, lz);
    int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    bool ok = i < p.nx && j < p.ny && k < L.kend;
    vox[3 * l] = ok ? grid_coord(p.ox, i, p.sx) : __longlong_as_double(0x7ff8000000000000ll);
    vox[3 * l + 1] = grid_coord(p.oy, j, p.sy);
    vox[3 * l + 2] = grid_coord(p.oz, k, p.sz);
  }
  for (int i = tid; i < NS * 16; i += blockDim.x) exw[i] = (i & 15) < 8 ? 0x7fffffff : -0x7fffffff;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], MODE == 6 ? 2 : 1);
      mbar_init(&empty[s], NCW);
      if (MODE == 6) mbar_init(reinterpret_cast<uint64_t*>(flag + 8) + s, 1);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (MODE >= 4 && warp == 0) {  // 512 TMEM columns (accumulators, or mode 6's windows)
    const unsigned a = (unsigned)__cvta_generic_to_shared(flag + 4);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // Transmit delay of every tile voxel for every angle (das.cpp:162), once.
  for (int i = tid; i < p.A * V; i += blockDim.x) {
    const int a = i / V, l = i % V;
    const AngleConst ac = p.ang[a];
    ttxA[i] = tx_delay(vox[3 * l], vox[3 * l + 2], ac.sina, ac.cosa, ac.ref, p.c);
  }
  __syncthreads();

  // The producers need few registers; the consumers hold VPW x J complex
  // accumulators (plus the row cache in mode 3).
  constexpr int kConsRegs = das2_cons_regs(NCW, PW);
  // (mode 0 with 4 producer warps fits the launch allocation and is faster
  // without the split)
  constexpr bool kSplit = (MODE >= 3 || PW > 4) && kConsRegs > das2_launch_regs(NCW + PW);
  if (warp >= NCW) {
    if (kSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(das2_prod_regs(PW, NCW)));
    // ============================ producers ============================
    // Per stage: (1) conservative per-element windows from the tile's bounding
    // box, TMA issued at once; (2) the exact FP64 table, computed while the
    // copy is in flight; (3) one arrival on full[] completes the stage when
    // both the table and the TMA bytes are in.
    const int tp = tid - NCW * 32;
    unsigned long long n_oow = 0, n_taps = 0;
    int stage = 0;
    const int nblk = (p.E + EB - 1) / EB;
    // Valid part of the tile's voxel box (for the window bounds).
    const int i1 = min(i0 + L.TX, p.nx) - 1, j1 = min(j0 + L.TY, p.ny) - 1,
              k1 = min(k0 + L.TZ, L.kend) - 1;
    const double bx0 = grid_coord(p.ox, i0, p.sx), bx1 = grid_coord(p.ox, i1, p.sx);
    const double by0 = grid_coord(p.oy, j0, p.sy), by1 = grid_coord(p.oy, j1, p.sy);
    const double bz0 = grid_coord(p.oz, k0, p.sz), bz1 = grid_coord(p.oz, k1, p.sz);
    // Tile transmit-delay range per angle (linear in p: box corners).
    for (int a = tp; a < p.A; a += NPT) {
      const AngleConst ac = p.ang[a];
      tbound[2 * a] = (fmin(bx0 * ac.sina, bx1 * ac.sina) + bz0 * ac.cosa - ac.ref) / p.c;
      tbound[2 * a + 1] = (fmax(bx0 * ac.sina, bx1 * ac.sina) + bz1 * ac.cosa - ac.ref) / p.c;
    }
    for (int eb = 0; eb < nblk; ++eb) {
      if (tp == 0) flag[0] = 0;
      named_sync(1, NPT);
#pragma unroll 1
      for (int b0 = 0; b0 < V * EB; b0 += NPT) {
        const int idx = b0 + tp;
        unsigned bits = 0;
        if (idx < V * EB) {
          int l = idx % V, el = idx / V, e = eb * EB + el;
          double v = -1.0;
          double px = vox[3 * l], py = vox[3 * l + 1], pz = vox[3 * l + 2];
          if (e < p.E && px == px) {
            double ex = __ldg(p.elem + 3 * e), ey = __ldg(p.elem + 3 * e + 1),
                   ez = __ldg(p.elem + 3 * e + 2);
            if (!(p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum))) {
              v = rx_delay(px, py, pz, ex, ey, ez, p.c);
              bits = 1u << el;
            }
          }
          rc[idx] = v;
        }
        // Elements with at least one voxel inside the aperture.
        bits = __reduce_or_sync(0xffffffffu, bits);
        if (lane == 0 && bits) atomicOr(&flag[0], (int)bits);
      }
      // Receive-range bounds of each element over the tile box.
      if (tp < EB && eb * EB + tp < p.E) {
        const int e = eb * EB + tp;
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
      named_sync(1, NPT);
      const int active = flag[0];
      if (!active) continue;

      for (int a = 0; a < p.A; ++a) {
        const int slot = stage % NS;
        if (L.hint) mbar_wait_hint(&empty[slot], ((stage / NS) & 1) ^ 1, L.hint); else mbar_wait(&empty[slot], ((stage / NS) & 1) ^ 1);
        SlotHdr& h = hdr[slot];
        const AngleConst ac = p.ang[a];
        // (1) lanes 0..EB-1 of the first producer warp: conservative window of
        //     element el (s = fs (ttx + |p - e|/c - t0), one row of margin),
        //     packing by an in-warp scan, and the element's TMA.  (With
        //     L.exactwin this runs after the table, on the exact tap range.)
        auto windows = [&](bool exact) {
          if (tp >= 32) return;
          int lo = 0x7fffffff, hi = kInactive, n = 0;
          if (tp < EB && ((active >> tp) & 1)) {
            if (exact) {
              const int* ew = exw + slot * 16;
              if (ew[tp] <= ew[8 + tp]) {
                lo = ew[tp];
                hi = ew[8 + tp];
                n = hi - lo + 2;
              }
            } else {
              const double smin = (tbound[2 * a] + dbound[2 * tp] - ac.t0) * p.fs;
              const double smax = (tbound[2 * a + 1] + dbound[2 * tp + 1] - ac.t0) * p.fs;
              const double flo = fmax(floor(smin) - 1.0, -1.0);
              const double fhi = fmin(floor(smax) + 1.0, (double)(p.T - 1));
              if (flo <= fhi) {
                lo = (int)flo;
                hi = (int)fhi;
                n = hi - lo + 2;
              }
            }
          }
          int pre = n;  // inclusive scan over lanes 0..EB-1
#pragma unroll
          for (int o = 1; o < EB; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, pre, o);
            if (tp >= o) pre += v;
          }
          if (MODE == 6 && n > 0) {
            // Whole time-row pairs: the slot starts on an even global row.
            const int r0 = (lo + 1) & ~1;
            n = ((hi + 3 - r0) + 1) & ~1;
            lo = r0 - 1;
          }
          if (MODE == 6) {  // the scan above ran on the unaligned sizes: redo it
            pre = n;
#pragma unroll
            for (int o = 1; o < EB; o <<= 1) {
              int v = __shfl_up_sync(0xffffffffu, pre, o);
              if (tp >= o) pre += v;
            }
          }
          const int base = pre - n;
          const bool fits = pre <= rslot;
          if (MODE == 6) {
            const int used = __reduce_max_sync(0xffffffffu, (tp < EB && n > 0 && fits) ? pre : 0);
            if (tp == 0) h.pad = used;
          }
          if (tp < EB) {
            h.wmin[tp] = lo;
            h.wmax[tp] = hi;
            h.wbase[tp] = n == 0 ? -2 : (fits ? base : -1);
            if (n > 0 && fits && !(L.debug & 2)) {
              const unsigned bytes = (unsigned)n * fpass * (unsigned)sizeof(float2);
              uint64_t* bar = MODE == 6 ? reinterpret_cast<uint64_t*>(flag + 8) + slot : &full[slot];
              unsigned b = (unsigned)__cvta_generic_to_shared(bar);
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(bytes)
                           : "memory");
              if (MODE == 6) {
                const size_t pair0 = ((size_t)a * p.E + (eb * EB + tp)) * (size_t)((p.T + 3) / 2) +
                                     (size_t)((lo + 1) / 2);
                bulk_g2s(win + (size_t)slot * wstride + (size_t)base * fpass,
                         iq + pair0 * 2 * fpass, bytes, bar);
              } else {
                size_t row0 = iq_row_index(p, a, eb * EB + tp, lo + 1);
                bulk_g2s(win + ((size_t)slot * rslot + base) * fpass, iq + row0 * fpass, bytes,
                         bar);
              }
            }
          }
          if (tp == 0) {
            h.done = 0;
            h.eb = eb;
            h.a = a;
          }
          if (exact && tp < EB) {  // reset for this slot's next use (ordered by (3))
            exw[slot * 16 + tp] = 0x7fffffff;
            exw[slot * 16 + 8 + tp] = -0x7fffffff;
          }
        };
        if (!L.exactwin) windows(false);
        // L2 prefetch of the window L.pf stages ahead (same bounds; the element
        // may be skipped later, so only elements whose aperture cone can reach
        // the tile box are prefetched).
        if (L.pf > 0 && tp < EB) {
          const int s2 = eb * p.A + a + L.pf;
          const int eb2 = s2 / p.A, a2 = s2 % p.A, e2 = eb2 * EB + tp;
          if (e2 < p.E) {
            const double ex = __ldg(p.elem + 3 * e2), ey = __ldg(p.elem + 3 * e2 + 1),
                         ez = __ldg(p.elem + 3 * e2 + 2);
            const double dxn = fmax(fmax(bx0 - ex, ex - bx1), 0.0);
            const double dyn = fmax(fmax(by0 - ey, ey - by1), 0.0);
            const double dzn = fmax(fmax(bz0 - ez, ez - bz1), 0.0);
            const bool reach = !(p.fnum > 0.0) ||
                               sqrt(dxn * dxn + dyn * dyn) <= (bz1 - ez) / (2.0 * p.fnum) + 1e-9;
            if (reach) {
              const double dxf = fmax(fabs(bx0 - ex), fabs(bx1 - ex));
              const double dyf = fmax(fabs(by0 - ey), fabs(by1 - ey));
              const double dzf = fmax(fabs(bz0 - ez), fabs(bz1 - ez));
              const AngleConst ac2 = p.ang[a2];
              const double smin =
                  (tbound[2 * a2] + sqrt(dxn * dxn + dyn * dyn + dzn * dzn) / p.c - ac2.t0) * p.fs;
              const double smax =
                  (tbound[2 * a2 + 1] + sqrt(dxf * dxf + dyf * dyf + dzf * dzf) / p.c - ac2.t0) *
                  p.fs;
              const double flo = fmax(floor(smin) - 1.0, -1.0);
              const double fhi = fmin(floor(smax) + 1.0, (double)(p.T - 1));
              if (flo <= fhi) {
                const unsigned bytes = (unsigned)((int)fhi - (int)flo + 2) * fpass * 8u;
                const float2* src = iq + iq_row_index(p, a2, e2, (int)flo + 1) * fpass;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes)
                             : "memory");
              }
            }
          }
        }
        // (2) exact table (das.cpp:159-197) while the bytes are in flight.
        const double* ttx = ttxA + (size_t)a * V;
        float4* t = tab + slot * EB * V;
        if (L.debug & 4) {  // diagnostic: table math skipped (first window row)
          named_sync(1, NPT);
          for (int idx = tp; idx < V * EB; idx += NPT) {
            const int el = idx / V;
            t[idx] = make_float4(__int_as_float(rc[idx] >= 0.0 ? h.wmin[el] + 1 : kInactive), 0.5f,
                                 1.f, 0.f);
          }
        } else
#pragma unroll 1
        for (int idx = tp; idx < V * EB; idx += NPT) {
          int l = idx % V;
          double r = rc[idx];
          float4 ent = make_float4(__int_as_float(kInactive), 0.f, 0.f, 0.f);
          if (r >= 0.0) {
            double tau = xadd(ttx[l], r);
            double s = xmul(xsub(tau, ac.t0), p.fs);
            int s0 = kInactive;
            float frac = 0.f;
            if (p.interp) {
              double sfl = floor(s);
              double fr = xsub(s, sfl);
              bool live0 = sfl >= 0.0 && sfl < (double)p.T;
              bool live1 = fr > 0.0 && xadd(sfl, 1.0) >= 0.0 && xadd(sfl, 1.0) < (double)p.T;
              if (live0 || live1) {
                s0 = (int)sfl;
                frac = (float)fr;
                n_taps += (int)live0 + (int)live1;
              } else {
                ++n_oow;
              }
            } else {
              double ri = round(s);
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
          t[idx] = ent;
          if (L.exactwin) {  // a warp's 32 entries belong to one element (V % 32 == 0)
            const int s0 = __float_as_int(ent.x);
            const int mn = __reduce_min_sync(0xffffffffu, s0 == kInactive ? 0x7fffffff : s0);
            const int mx = __reduce_max_sync(0xffffffffu, s0 == kInactive ? -0x7fffffff : s0);
            if (lane == 0 && mn <= mx) {
              atomicMin(exw + slot * 16 + idx / V, mn);
              atomicMax(exw + slot * 16 + 8 + idx / V, mx);
            }
          }
        }
        // (3) table done on every producer thread -> one arrival completes
        // the phase together with the TMA bytes.
        named_sync(1, NPT);
        if (L.exactwin) windows(true);
        if (MODE == 6 && tp == 0) {
          // Staged rows -> TMEM: lane = frame (two 128-frame groups), column
          // 2 x (row in slot) + re/im.  One tcgen05.cp.128x256b moves two
          // time-row pairs of 128 frames; commit arrives on full[slot].
          uint64_t* sbar = reinterpret_cast<uint64_t*>(flag + 8) + slot;
          mbar_arrive(sbar);
          mbar_wait(sbar, (stage / NS) & 1);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(win + (size_t)slot * wstride);
          const uint32_t tcol = (uint32_t)flag[4] + (uint32_t)(slot * 256);
          const int pairs = h.pad / 2;
          const uint32_t lbo = (uint32_t)fpass * 16u;
          for (int g = 0; g * 128 < fpass; ++g)
            for (int k = 0; 2 * k < pairs; ++k) {
              const uint32_t sa = sbase + (uint32_t)(2 * k) * lbo + (uint32_t)g * 2048u;
              const uint64_t d = (uint64_t)((sa >> 4) & 0x3FFF) |
                                 ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                                 ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
              asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(
                               tcol + (uint32_t)(g * 128 + 8 * k)),
                           "l"(d));
            }
          unsigned b = (unsigned)__cvta_generic_to_shared(&full[slot]);
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
              : "memory");
        }
        if (tp == 0) mbar_arrive(&full[slot]);
        ++stage;
      }
    }
    // Termination stage.
    const int slot = stage % NS;
    if (L.hint) mbar_wait_hint(&empty[slot], ((stage / NS) & 1) ^ 1, L.hint); else mbar_wait(&empty[slot], ((stage / NS) & 1) ^ 1);
    if (tp == 0) {
      hdr[slot].done = 1;
      mbar_arrive(&full[slot]);
      if (MODE == 6) mbar_arrive(&full[slot]);
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
    return;
  }

  // ============================== consumers ==============================
  if (kSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsRegs));
  if (MODE == 0) {
    const int half = lane >> 4, l16 = lane & 15;
    // Voxel of (vp, half).  With L.pairy the half-warp partners are
    // y-neighbours: the y component of the receive delay changes by < 1
    // sample per voxel, so most partners hit the same IQ rows and the warp's
    // two 128 B half-rows coincide (one shared-memory wavefront, broadcast).
    int lv[VPW];
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      const int q = warp * VPW + vp;
      const int lx = q % L.TX, yp = (q / L.TX) % (L.TY >> 1), lz = q / (L.TX * (L.TY >> 1));
      // pairy 2 (diagonal): warp w takes voxel (x = (w + m) % TX, row m) for
      // its m-th voxel, so every warp samples every row and column of the
      // tile and the aperture boundary loads the warps evenly (needs
      // NCW == TX and 2 VPW rows).
      const int m = vp * 2 + half;
      lv[vp] = L.pairy == 2   ? (warp + m) % L.TX + L.TX * m
               : L.pairy == 1 ? lx + L.TX * (2 * yp + half + L.TY * lz)
                              : q * 2 + half;
    }
    float2 acc[VPW][J];
#pragma unroll
    for (int v = 0; v < VPW; ++v)
#pragma unroll
      for (int j = 0; j < J; ++j) acc[v][j] = make_float2(0.f, 0.f);

    for (int stage = 0;; ++stage) {
      const int slot = stage % NS;
      if (L.hint) mbar_wait_hint(&full[slot], (stage / NS) & 1, L.hint); else mbar_wait(&full[slot], (stage / NS) & 1);
      const SlotHdr& h = hdr[slot];
      if (h.done) break;
      const float4* t = tab + slot * EB * V;
      const float2* w = win + (size_t)slot * rslot * fpass;
      for (int el = 0; el < EB && !(L.debug & 1); ++el) {
        const int wb = h.wbase[el];
        if (wb == -2) continue;
        if (wb >= 0) {
          const int row_off = wb - h.wmin[el];
#pragma unroll
          for (int vp = 0; vp < VPW; ++vp) {
            const int l = lv[vp];
            const float4 ent = t[el * V + l];
            const int s0 = __float_as_int(ent.x);
            if (s0 != kInactive)
              gather_taps<J>(w + (size_t)(row_off + s0) * fpass + l16, fpass, ent, acc[vp]);
          }
        } else {
          const float2* g = iq + (iq_row_index(p, h.a, h.eb * EB + el, 0) + 1) * fpass + l16;
#pragma unroll
          for (int vp = 0; vp < VPW; ++vp) {
            const int l = lv[vp];
            const float4 ent = t[el * V + l];
            const int s0 = __float_as_int(ent.x);
            if (s0 != kInactive) gather_taps<J>(g + (ptrdiff_t)s0 * fpass, fpass, ent, acc[vp]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    const float inv = (float)(1.0 / p.A);
    const size_t N = (size_t)p.nx * p.ny * p.nz;
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      const int l = lv[vp];
      int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
      int i = i0 + lx, j = j0 + ly, k = k0 + lz;
      if (i < p.nx && j < p.ny && k < L.kend) {
        size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          int f = L.pass * fpass + 16 * jj + l16;
          if (f < p.F)
            x[(size_t)f * N + flat] = make_float2(acc[vp][jj].x * inv, acc[vp][jj].y * inv);
        }
      }
    }
  } else if (MODE == 4) {
    // Mode 3's lane mapping (half-warp y-columns, warp-uniform row reloads),
    // with the accumulators in tensor memory instead of registers: per
    // (voxel, element) tcgen05.ld the voxel's 2J fp32 sums, FMA, tcgen05.st.
    // The freed registers allow 16 consumer warps.  Warp w uses lanes of
    // quadrant w % 4 and columns [(w / 4) VPW 32, + VPW 32).
    const int half = lane >> 4, l16 = lane & 15;
    const int lbase = (warp * 2 + half) * VPW;
    constexpr int kNone = -0x40000000;
    constexpr int NC = 2 * J;
    const uint32_t tbase = (uint32_t)flag[4] + ((uint32_t)(32 * (warp & 3)) << 16) +
                           (uint32_t)((warp >> 2) * VPW * 32);
    {
      uint32_t z[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) z[c] = 0u;
#pragma unroll
      for (int vp = 0; vp < VPW; ++vp) tm_st<NC>(tbase + 32 * vp, z);
    }

    for (int stage = 0;; ++stage) {
      const int slot = stage % NS;
      mbar_wait(&full[slot], (stage / NS) & 1);
      const SlotHdr& h = hdr[slot];
      if (h.done) break;
      const float4* t = tab + slot * EB * V + lbase;
      const float2* w = win + (size_t)slot * rslot * fpass;
      for (int el = 0; el < EB && !(L.debug & 1); ++el) {
        const int wb = h.wbase[el];
        if (wb == -2) continue;
        const float2* base =
            wb >= 0 ? w + (ptrdiff_t)(wb - h.wmin[el]) * fpass + l16
                    : iq + (iq_row_index(p, h.a, h.eb * EB + el, 0) + 1) * fpass + l16;
        const int srow = wb >= 0 ? h.wmin[el] + 1 : 0;  // a row inside the window
        float2 c0[J], dd[J];
        int cur = kNone;
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) {
          const float4 ent = t[el * V + vp];
          const int s0 = __float_as_int(ent.x);
          const bool act = s0 != kInactive;
          if (!__any_sync(0xffffffffu, act)) continue;
          uint32_t ra[NC];
          tm_wait_st();
          tm_ld<NC>(tbase + 32 * vp, ra);
          const int se = act ? s0 : (cur != kNone ? cur : srow);
          if (__any_sync(0xffffffffu, se != cur)) {
            cur = se;
            const float2* r0 = base + (ptrdiff_t)se * fpass;
#pragma unroll
            for (int j = 0; j < J; ++j) {
              const float2 x0 = r0[16 * j], x1 = r0[fpass + 16 * j];
              c0[j] = x0;
              dd[j] = make_float2(x1.x - x0.x, x1.y - x0.y);
            }
          }
          const float fr = ent.y, cr = act ? ent.z : 0.f, ci = act ? ent.w : 0.f;
          tm_wait_ld();
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const float vr = fmaf(fr, dd[j].x, c0[j].x), vi = fmaf(fr, dd[j].y, c0[j].y);
            ra[2 * j] = __float_as_uint(fmaf(cr, vr, fmaf(-ci, vi, __uint_as_float(ra[2 * j]))));
            ra[2 * j + 1] =
                __float_as_uint(fmaf(cr, vi, fmaf(ci, vr, __uint_as_float(ra[2 * j + 1]))));
          }
          tm_st<NC>(tbase + 32 * vp, ra);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    const float inv = (float)(1.0 / p.A);
    const size_t N = (size_t)p.nx * p.ny * p.nz;
    tm_wait_st();
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      uint32_t ra[NC];
      tm_ld<NC>(tbase + 32 * vp, ra);
      tm_wait_ld();
      int lx, ly, lz;
      tile_local<MODE>(lbase + vp, L, lx, ly, lz);
      int i = i0 + lx, j = j0 + ly, k = k0 + lz;
      if (i < p.nx && j < p.ny && k < L.kend) {
        size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          int f = L.pass * fpass + 16 * jj + l16;
          if (f < p.F)
            x[(size_t)f * N + flat] = make_float2(__uint_as_float(ra[2 * jj]) * inv,
                                                  __uint_as_float(ra[2 * jj + 1]) * inv);
        }
      }
    }
    // All consumer warps are done with TMEM -> warp 0 frees it.
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    named_sync(2, NCW * 32);
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(flag[4]));
    }
  } else if (MODE == 6) {
    // Lanes = frames: warp w reads TMEM lane quadrant q = w % 4, i.e. frames
    // g 128 + 32 q + lane of frame group g, for the voxels
    // {sub, sub + NSUB, ...} (sub = w / 4).  Per voxel and element one
    // tcgen05.ld.32x32b.x4 at column 2 (slot row of s0) returns x0 and x1 of
    // 32 frames; everything is warp-uniform (one voxel per warp at a time).
    constexpr int NSUB = NCW / 4;
    constexpr int G = (16 * J + 127) / 128;
    const int q = warp & 3, sub = warp >> 2;
    const int nf = min(fpass, p.F - L.pass * fpass);
    const uint32_t tlane = (uint32_t)flag[4] + ((uint32_t)(32 * q) << 16);
    const size_t npair = (size_t)((p.T + 3) / 2);
    float2 acc[VPW][G];
#pragma unroll
    for (int v = 0; v < VPW; ++v)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[v][g] = make_float2(0.f, 0.f);

    for (int stage = 0;; ++stage) {
      const int slot = stage % NS;
      mbar_wait(&full[slot], (stage / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const SlotHdr& h = hdr[slot];
      if (h.done) break;
      const float4* t = tab + slot * EB * V + sub;
      for (int el = 0; el < EB && !(L.debug & 1); ++el) {
        const int wb = h.wbase[el];
        if (wb == -2) continue;
        if (wb < 0) {  // window did not fit: taps from global memory (pair layout)
          const float2* g0 = iq + ((size_t)h.a * p.E + (h.eb * EB + el)) * npair * 2 * fpass;
#pragma unroll
          for (int vp = 0; vp < VPW; ++vp) {
            const float4 ent = t[el * V + vp * NSUB];
            const int s0 = __float_as_int(ent.x);
            if (s0 == kInactive) continue;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const int fl = g * 128 + 32 * q + lane;
              if (fl < nf) {
                const int r = s0 + 1;
                const float2 x0 = g0[((size_t)(r >> 1) * fpass + fl) * 2 + (r & 1)];
                const float2 x1 = g0[((size_t)((r + 1) >> 1) * fpass + fl) * 2 + ((r + 1) & 1)];
                const float vr = fmaf(ent.y, x1.x - x0.x, x0.x), vi = fmaf(ent.y, x1.y - x0.y, x0.y);
                acc[vp][g].x = fmaf(ent.z, vr, fmaf(-ent.w, vi, acc[vp][g].x));
                acc[vp][g].y = fmaf(ent.z, vi, fmaf(ent.w, vr, acc[vp][g].y));
              }
            }
          }
          continue;
        }
        const uint32_t cb = tlane + (uint32_t)(slot * 256) + 2u * (uint32_t)(wb - h.wmin[el]);
        constexpr int NB6 = 8;  // voxels whose taps are in flight per tcgen05.wait::ld
#pragma unroll
        for (int vb = 0; vb < VPW; vb += NB6) {
          float4 ent[NB6];
          uint32_t r[NB6][G][4];
#pragma unroll
          for (int b = 0; b < NB6; ++b) ent[b] = t[el * V + (vb + b) * NSUB];
          // Unconditional loads (no divergence around the .sync.aligned
          // instructions): an inactive voxel reads a staged row with zero weight.
#pragma unroll
          for (int b = 0; b < NB6; ++b) {
            const int s0 = __float_as_int(ent[b].x);
            const int sr = s0 == kInactive ? h.wmin[el] : s0;  // a staged row
#pragma unroll
            for (int g = 0; g < G; ++g)
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(r[b][g][0]), "=r"(r[b][g][1]), "=r"(r[b][g][2]), "=r"(r[b][g][3])
                           : "r"(cb + (uint32_t)(g * 128 + 2 * sr)));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int b = 0; b < NB6; ++b) {
            const bool act = __float_as_int(ent[b].x) != kInactive;
            const float fr = ent[b].y, cr = act ? ent[b].z : 0.f, ci = act ? ent[b].w : 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              {
                const float x0r = __uint_as_float(r[b][g][0]), x0i = __uint_as_float(r[b][g][1]);
                const float x1r = __uint_as_float(r[b][g][2]), x1i = __uint_as_float(r[b][g][3]);
                const float vr = fmaf(fr, x1r - x0r, x0r), vi = fmaf(fr, x1i - x0i, x0i);
                acc[vb + b][g].x = fmaf(cr, vr, fmaf(-ci, vi, acc[vb + b][g].x));
                acc[vb + b][g].y = fmaf(cr, vi, fmaf(ci, vr, acc[vb + b][g].y));
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    const float inv = (float)(1.0 / p.A);
    const size_t N = (size_t)p.nx * p.ny * p.nz;
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      int lx, ly, lz;
      tile_local<MODE>(vp * NSUB + sub, L, lx, ly, lz);
      int i = i0 + lx, j = j0 + ly, k = k0 + lz;
      if (i < p.nx && j < p.ny && k < L.kend) {
        size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int fl = g * 128 + 32 * q + lane;
          if (fl < nf)
            x[(size_t)(L.pass * fpass + fl) * N + flat] =
                make_float2(acc[vp][g].x * inv, acc[vp][g].y * inv);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    named_sync(2, NCW * 32);
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(flag[4]));
    }
  } else if (MODE == 5) {
    // Mode 4 with packed FP32 arithmetic (fma.rn.f32x2 / FFMA2): per sample
    //   v = x0 + fr (x1 - x0),  P += cr v,  Q += ci v      (3 FFMA2)
    // and acc = (P.x - Q.y, P.y + Q.x) at the end -- the same products as
    // acc += (cr + i ci) v, summed as two pairs.  P and Q (4 J fp32 per voxel)
    // live in TMEM: warp w, lanes of quadrant w % 4, columns
    // [(w / 4) VPW 4 J, + VPW 4 J).
    const int half = lane >> 4, l16 = lane & 15;
    const int lbase = (warp * 2 + half) * VPW;
    constexpr int kNone = -0x40000000;
    constexpr int NC = 4 * J;
    const uint32_t tbase = (uint32_t)flag[4] + ((uint32_t)(32 * (warp & 3)) << 16) +
                           (uint32_t)((warp >> 2) * VPW * NC);
    {
      uint32_t z[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) z[c] = 0u;
#pragma unroll
      for (int vp = 0; vp < VPW; ++vp) tm_st<NC>(tbase + NC * vp, z);
    }
    const unsigned long long kM1 = f2bc(-1.f);

    for (int stage = 0;; ++stage) {
      const int slot = stage % NS;
      mbar_wait(&full[slot], (stage / NS) & 1);
      const SlotHdr& h = hdr[slot];
      if (h.done) break;
      const float4* t = tab + slot * EB * V + lbase;
      const float2* w = win + (size_t)slot * rslot * fpass;
      for (int el = 0; el < EB && !(L.debug & 1); ++el) {
        const int wb = h.wbase[el];
        if (wb == -2) continue;
        const float2* base =
            wb >= 0 ? w + (ptrdiff_t)(wb - h.wmin[el]) * fpass + l16
                    : iq + (iq_row_index(p, h.a, h.eb * EB + el, 0) + 1) * fpass + l16;
        const int srow = wb >= 0 ? h.wmin[el] + 1 : 0;  // a row inside the window
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(w) +
                               (uint32_t)((wb - h.wmin[el]) * fpass + l16) * 8u;
        unsigned long long c0[J], dd[J];
        int cur = kNone;
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) {
          const float4 ent = t[el * V + vp];
          const int s0 = __float_as_int(ent.x);
          const bool act = s0 != kInactive;
          if (!__any_sync(0xffffffffu, act)) continue;
          uint32_t ra[NC];
          tm_wait_st();
          tm_ld<NC>(tbase + NC * vp, ra);
          const int se = act ? s0 : (cur != kNone ? cur : srow);
          if (__any_sync(0xffffffffu, se != cur)) {
            cur = se;
            if (wb >= 0) {  // the window row in shared memory: 32-bit LDS addressing
              const uint32_t r0 = sbase + (uint32_t)(se * fpass) * 8u;
#pragma unroll
              for (int j = 0; j < J; ++j) {
                unsigned long long x0, x1;
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x0) : "r"(r0 + 128u * j));
                asm volatile("ld.shared.b64 %0, [%1];"
                             : "=l"(x1)
                             : "r"(r0 + (uint32_t)fpass * 8u + 128u * j));
                c0[j] = x0;
                dd[j] = ffma2(x0, kM1, x1);  // x1 - x0
              }
            } else {
              const unsigned long long* r0 =
                  reinterpret_cast<const unsigned long long*>(base + (ptrdiff_t)se * fpass);
#pragma unroll
              for (int j = 0; j < J; ++j) {
                const unsigned long long x0 = r0[16 * j], x1 = r0[fpass + 16 * j];
                c0[j] = x0;
                dd[j] = ffma2(x0, kM1, x1);
              }
            }
          }
          const unsigned long long fr = f2bc(ent.y), cr = f2bc(act ? ent.z : 0.f),
                                   ci = f2bc(act ? ent.w : 0.f);
          tm_wait_ld();
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const unsigned long long v = ffma2(fr, dd[j], c0[j]);
            const unsigned long long P = ffma2(cr, v, f2pk(ra[2 * j], ra[2 * j + 1]));
            const unsigned long long Q =
                ffma2(ci, v, f2pk(ra[2 * J + 2 * j], ra[2 * J + 2 * j + 1]));
            f2upk(P, ra[2 * j], ra[2 * j + 1]);
            f2upk(Q, ra[2 * J + 2 * j], ra[2 * J + 2 * j + 1]);
          }
          tm_st<NC>(tbase + NC * vp, ra);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    const float inv = (float)(1.0 / p.A);
    const size_t N = (size_t)p.nx * p.ny * p.nz;
    tm_wait_st();
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      uint32_t ra[NC];
      tm_ld<NC>(tbase + NC * vp, ra);
      tm_wait_ld();
      int lx, ly, lz;
      tile_local<MODE>(lbase + vp, L, lx, ly, lz);
      int i = i0 + lx, j = j0 + ly, k = k0 + lz;
      if (i < p.nx && j < p.ny && k < L.kend) {
        size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          int f = L.pass * fpass + 16 * jj + l16;
          const float re = __uint_as_float(ra[2 * jj]) - __uint_as_float(ra[2 * J + 2 * jj + 1]);
          const float im = __uint_as_float(ra[2 * jj + 1]) + __uint_as_float(ra[2 * J + 2 * jj]);
          if (f < p.F) x[(size_t)f * N + flat] = make_float2(re * inv, im * inv);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    named_sync(2, NCW * 32);
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(flag[4]));
    }
  } else if (MODE == 3) {
    // Half-warp h of warp w owns the y-column [(2w + h) VPW, (2w + h + 1) VPW)
    // of table entries; lanes = 16 frames.  The two halves reload their tap
    // rows together (warp-uniform branch) when either column's tap index
    // changes; a voxel outside the aperture gets zero weight on a valid row.
    const int half = lane >> 4, l16 = lane & 15;
    const int lbase = (warp * 2 + half) * VPW;
    constexpr int kNone = -0x40000000;
    float2 acc[VPW][J];
#pragma unroll
    for (int v = 0; v < VPW; ++v)
#pragma unroll
      for (int j = 0; j < J; ++j) acc[v][j] = make_float2(0.f, 0.f);

    for (int stage = 0;; ++stage) {
      const int slot = stage % NS;
      mbar_wait(&full[slot], (stage / NS) & 1);
      const SlotHdr& h = hdr[slot];
      if (h.done) break;
      const float4* t = tab + slot * EB * V + lbase;
      const float2* w = win + (size_t)slot * rslot * fpass;
      for (int el = 0; el < EB && !(L.debug & 1); ++el) {
        const int wb = h.wbase[el];
        if (wb == -2) continue;
        float4 ent[VPW];
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) ent[vp] = t[el * V + vp];
        if (wb < 0) {  // window did not fit the slot: straight from global memory
          const float2* g = iq + (iq_row_index(p, h.a, h.eb * EB + el, 0) + 1) * fpass + l16;
#pragma unroll
          for (int vp = 0; vp < VPW; ++vp) {
            const int s0 = __float_as_int(ent[vp].x);
            if (s0 != kInactive) gather_taps<J>(g + (ptrdiff_t)s0 * fpass, fpass, ent[vp], acc[vp]);
          }
          continue;
        }
        const float2* base = w + (ptrdiff_t)(wb - h.wmin[el]) * fpass + l16;
        const int srow = h.wmin[el] + 1;  // a row inside the window
        float2 c0[J], dd[J];
        int cur = kNone;
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) {
          const int s0 = __float_as_int(ent[vp].x);
          const bool act = s0 != kInactive;
          if (!__any_sync(0xffffffffu, act)) continue;
          const int se = act ? s0 : (cur != kNone ? cur : srow);
          if (__any_sync(0xffffffffu, se != cur)) {
            cur = se;
            const float2* r0 = base + (ptrdiff_t)se * fpass;
#pragma unroll
            for (int j = 0; j < J; ++j) {
              const float2 x0 = r0[16 * j], x1 = r0[fpass + 16 * j];
              c0[j] = x0;
              dd[j] = make_float2(x1.x - x0.x, x1.y - x0.y);
            }
          }
          const float fr = ent[vp].y, cr = act ? ent[vp].z : 0.f, ci = act ? ent[vp].w : 0.f;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const float vr = fmaf(fr, dd[j].x, c0[j].x), vi = fmaf(fr, dd[j].y, c0[j].y);
            acc[vp][j].x = fmaf(cr, vr, fmaf(-ci, vi, acc[vp][j].x));
            acc[vp][j].y = fmaf(cr, vi, fmaf(ci, vr, acc[vp][j].y));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    const float inv = (float)(1.0 / p.A);
    const size_t N = (size_t)p.nx * p.ny * p.nz;
#pragma unroll
    for (int vp = 0; vp < VPW; ++vp) {
      int lx, ly, lz;
      tile_local<MODE>(lbase + vp, L, lx, ly, lz);
      int i = i0 + lx, j = j0 + ly, k = k0 + lz;
      if (i < p.nx && j < p.ny && k < L.kend) {
        size_t flat = (size_t)i + (size_t)p.nx * ((size_t)j + (size_t)p.ny * k);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          int f = L.pass * fpass + 16 * jj + l16;
          if (f < p.F) x[(size_t)f * N + flat] = make_float2(acc[vp][jj].x * inv, acc[vp][jj].y * inv);
        }
      }
    }
  }
}

// Shared memory besides the NS window slots.
inline size_t das2_aux_smem(int V, int EB, int NS, int A) {
  return (size_t)NS * EB * V * 16 + (size_t)EB * V * 8 + (size_t)V * 24 + (size_t)A * V * 8 +
         (size_t)A * 16 + (size_t)EB * 16 + NS * sizeof(SlotHdr) + 2 * NS * 8 + 64 + NS * 64;
}

}  // namespace fqfg
