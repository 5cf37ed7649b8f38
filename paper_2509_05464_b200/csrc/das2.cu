// das2.cu -- 3D plane-wave delay-and-sum with coherent angle compounding:
// the warp-specialised, double-buffered production kernel.
//
// Semantics: das_reconstruct (proj/src/beamform/das.cpp:224-356) with the
// delay matrix of build_delay_matrix (das.cpp:126-208) evaluated on the fly:
//   mask   hypot(p.x-e.x, p.y-e.y) * 2 F# > p.z - e.z  -> skip   (das.cpp:165-168)
//   delay  tau = (p.x sin a + p.z cos a - min_n x_n sin a)/c + |p - e|/c
//   taps   s = (tau - t0) fs; linear: floor(s) w/ (1-frac), floor(s)+1 w/ frac
//          (only if frac > 0), each only inside [0, T); nearest: round(s)
//   value  weight * exp(+i 2 pi f_c tau), summed over elements, then over
//          angles, times 1/A (das.cpp:309-328).
//
// The delay of a (voxel, element, angle) triple does not depend on the frame,
// so the kernel is frames-innermost: one CTA owns a voxel tile and the 16 J
// frames of one pass, and the IQ layout [angle][element][row][frame] makes an
// element's time window over the tile one contiguous byte range.
//
//   producer warps (PW)   per stage s = (element block eb, angle a):
//     wait empty[s%NS]; conservative per-element windows from the tile box,
//     one elected lane per element issues a 1-D TMA bulk copy (cp.async.bulk)
//     completing on full[s%NS]; then the exact FP64 tap index / weight /
//     carrier rotation of every (voxel, element) -> table slot (overlapping
//     the copy).
//   consumer warps (NCW)  per stage: wait full[s%NS]; gather the two taps of
//     every (voxel, element, frame) from shared memory (lanes = 16 frames x 2
//     voxels, conflict-free 128 B half-warp rows), interpolate, rotate,
//     accumulate in registers (acc[VPW][J] complex f32); arrive empty[s%NS].
//
// NS = 2 slots, so the TMA copy and the FP64 table of stage s+1 run while the
// consumers gather stage s.  Elements whose window does not fit the slot are
// gathered straight from global memory (same arithmetic).  Measurements of
// this design and of the variants it beat are in profiles/r01_das2_C.md.
#include "common.cuh"

namespace fqfg {

constexpr int kInactive = (int)0x80000000;

FQFG_DEVICE void mbar_init(uint64_t* bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

FQFG_DEVICE void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

// Wait with back-off: a warp whose barrier is not ready sleeps `ns` between
// probes instead of re-issuing try_wait (das_tc's idle roles).
FQFG_DEVICE void mbar_wait_sleep(uint64_t* bar, unsigned phase, unsigned ns) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  while (true) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}

FQFG_DEVICE void mbar_arrive(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

FQFG_DEVICE void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

FQFG_DEVICE void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Two-tap interpolation, carrier rotation and accumulation for J frames:
// acc += rot * (x0 + frac (x1 - x0)), i.e. (1-frac) rot x0 + frac rot x1.
template <int J>
FQFG_DEVICE void gather_taps(const float2* r0, int fpass, const float4 ent, float2 (&acc)[J]) {
  const float fr = ent.y, cr = ent.z, ci = ent.w;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    float2 x0 = r0[16 * j];
    float2 x1 = r0[fpass + 16 * j];
    float vr = fmaf(fr, x1.x - x0.x, x0.x);
    float vi = fmaf(fr, x1.y - x0.y, x0.y);
    acc[j].x = fmaf(cr, vr, fmaf(-ci, vi, acc[j].x));
    acc[j].y = fmaf(cr, vi, fmaf(ci, vr, acc[j].y));
  }
}

struct DasLaunch {
  int TX, TY, TZ;  // voxel tile
  int tiles_x, tiles_y;
  int kbeg, kend;  // z-slab
  int pass;
  int rcap;        // window rows per shared-memory slot
  long long x_v0;  // x holds voxels [x_v0, x_v0 + x_n) of the grid (a slab)
  long long x_n;
  unsigned long long* kblocks;      // das_tc: += MMA K blocks issued (instrumentation; may be null)
};

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

struct SlotHdr {
  int done, eb, a, pad;
  int wbase[8];  // >= 0 row in slot buffer, -1 gather from global, -2 element unused
  int wmin[8];
  int wmax[8];
};

// Consumer lane mapping (V = 2 NCW VPW voxels per tile, x fastest): lanes =
// 16 frames x 2 voxels (half-warps), fpass = 16 J; each voxel reads its two
// tap rows.
template <int J, int VPW, int NCW, int EB, int NS, int PW>
__global__ void __launch_bounds__((NCW + PW) * 32, 1)
    das2_kernel(const DasParams p, const DasLaunch L, const float2* __restrict__ iq,
                float2* __restrict__ x, unsigned long long* __restrict__ counters) {
  constexpr int V = NCW * VPW * 2;
  constexpr int NPT = PW * 32;
  static_assert(PW % 4 == 0 && NCW % 4 == 0, "setmaxnreg acts on whole warpgroups");
  static_assert(EB <= 8, "SlotHdr holds 8 elements");
  const int fpass = 16 * J;
  const int rslot = L.rcap;  // rows per slot

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* win = reinterpret_cast<float2*>(smem_raw);  // [NS][rslot][fpass]
  unsigned char* sp = smem_raw + (size_t)NS * rslot * fpass * sizeof(float2);
  float4* tab = reinterpret_cast<float4*>(sp);                // [NS][EB][V]
  double* rc = reinterpret_cast<double*>(tab + NS * EB * V);  // [EB][V]
  double* vox = rc + EB * V;                                  // [V][3]
  double* ttxA = vox + 3 * V;                                 // [A][V] transmit delays
  double* tbound = ttxA + (size_t)p.A * V;                    // [A][2] tile min/max ttx
  double* dbound = tbound + 2 * p.A;                          // [EB][2] |p-e|/c min/max
  SlotHdr* hdr = reinterpret_cast<SlotHdr*>(dbound + 2 * EB);  // [NS]
  uint64_t* full = reinterpret_cast<uint64_t*>(hdr + NS);
  uint64_t* empty = full + NS;
  int* flag = reinterpret_cast<int*>(empty + NS);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  int tile = blockIdx.x;
  const int tx = tile % L.tiles_x;
  tile /= L.tiles_x;
  const int ty = tile % L.tiles_y;
  // Deep planes first: deep tiles see more elements inside the f-number cone
  // and cost more, so the cheap shallow tiles fill the last wave.
  const int ntz = (L.kend - L.kbeg + L.TZ - 1) / L.TZ;
  const int tz = ntz - 1 - tile / L.tiles_y;
  const int i0 = tx * L.TX, j0 = ty * L.TY, k0 = L.kbeg + tz * L.TZ;

  for (int l = tid; l < V; l += blockDim.x) {
    const int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
    int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    bool ok = i < p.nx && j < p.ny && k < L.kend;
    vox[3 * l] = ok ? grid_coord(p.ox, i, p.sx) : __longlong_as_double(0x7ff8000000000000ll);
    vox[3 * l + 1] = grid_coord(p.oy, j, p.sy);
    vox[3 * l + 2] = grid_coord(p.oz, k, p.sz);
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // Transmit delay of every tile voxel for every angle (das.cpp:162), once.
  for (int i = tid; i < p.A * V; i += blockDim.x) {
    const int a = i / V, l = i % V;
    const AngleConst ac = p.ang[a];
    ttxA[i] = tx_delay(vox[3 * l], vox[3 * l + 2], ac.sina, ac.cosa, ac.ref, p.c);
  }
  __syncthreads();

  // The producers need few registers; the consumers hold VPW x J complex
  // accumulators.
  constexpr int kConsRegs = das2_cons_regs(NCW, PW);
  // (4 producer warps fit the launch allocation and are faster without the split)
  constexpr bool kSplit = PW > 4 && kConsRegs > das2_launch_regs(NCW + PW);
  if (warp >= NCW) {
    if (kSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(das2_prod_regs(PW, NCW)));
    // ============================ producers ============================
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
        mbar_wait(&empty[slot], ((stage / NS) & 1) ^ 1);
        SlotHdr& h = hdr[slot];
        const AngleConst ac = p.ang[a];
        // (1) lanes 0..EB-1 of the first producer warp: conservative window of
        //     element el (s = fs (ttx + |p - e|/c - t0), one row of margin),
        //     packing by an in-warp scan, and the element's TMA.
        if (tp < 32) {
          int lo = 0x7fffffff, hi = kInactive, n = 0;
          if (tp < EB && ((active >> tp) & 1)) {
            const double smin = (tbound[2 * a] + dbound[2 * tp] - ac.t0) * p.fs;
            const double smax = (tbound[2 * a + 1] + dbound[2 * tp + 1] - ac.t0) * p.fs;
            // clamped to the stored rows [iq_row0, iq_row0 + iq_rows): the tile
            // box's far corner can lie outside the f-number cone that bounds
            // every live tap (slab_rows), and those rows are never read
            const double flo = fmax(floor(smin) - 1.0, fmax(-1.0, (double)(p.iq_row0 - 1)));
            const double fhi = fmin(floor(smax) + 1.0,
                                    fmin((double)(p.T - 1), (double)(p.iq_row0 + p.iq_rows - 3)));
            if (flo <= fhi) {
              lo = (int)flo;
              hi = (int)fhi;
              n = hi - lo + 2;
            }
          }
          int pre = n;  // inclusive scan over lanes 0..EB-1
#pragma unroll
          for (int o = 1; o < EB; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, pre, o);
            if (tp >= o) pre += v;
          }
          const int base = pre - n;
          const bool fits = pre <= rslot;
          if (tp < EB) {
            h.wmin[tp] = lo;
            h.wmax[tp] = hi;
            h.wbase[tp] = n == 0 ? -2 : (fits ? base : -1);
            if (n > 0 && fits) {
              const unsigned bytes = (unsigned)n * fpass * (unsigned)sizeof(float2);
              unsigned b = (unsigned)__cvta_generic_to_shared(&full[slot]);
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(bytes)
                           : "memory");
              const long long row0 = iq_row_index(p, a, eb * EB + tp, lo + 1);
              bulk_g2s(win + ((size_t)slot * rslot + base) * fpass, iq + row0 * fpass, bytes,
                       &full[slot]);
            }
          }
          if (tp == 0) {
            h.done = 0;
            h.eb = eb;
            h.a = a;
          }
        }
        // (2) exact table (das.cpp:159-197) while the bytes are in flight.
        const double* ttx = ttxA + (size_t)a * V;
        float4* t = tab + slot * EB * V;
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
        }
        // (3) table done on every producer thread -> one arrival completes
        // the phase together with the TMA bytes.
        named_sync(1, NPT);
        if (tp == 0) mbar_arrive(&full[slot]);
        ++stage;
      }
    }
    // Termination stage.
    const int slot = stage % NS;
    mbar_wait(&empty[slot], ((stage / NS) & 1) ^ 1);
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
    return;
  }

  // ============================== consumers ==============================
  if (kSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsRegs));
  const int half = lane >> 4, l16 = lane & 15;
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
    const float4* t = tab + slot * EB * V;
    const float2* w = win + (size_t)slot * rslot * fpass;
    for (int el = 0; el < EB; ++el) {
      const int wb = h.wbase[el];
      if (wb == -2) continue;
      if (wb >= 0) {
        const int row_off = wb - h.wmin[el];
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) {
          const int l = (warp * VPW + vp) * 2 + half;
          const float4 ent = t[el * V + l];
          const int s0 = __float_as_int(ent.x);
          if (s0 != kInactive)
            gather_taps<J>(w + (size_t)(row_off + s0) * fpass + l16, fpass, ent, acc[vp]);
        }
      } else {
        const float2* g = iq + (iq_row_index(p, h.a, h.eb * EB + el, 0) + 1) * fpass + l16;
#pragma unroll
        for (int vp = 0; vp < VPW; ++vp) {
          const int l = (warp * VPW + vp) * 2 + half;
          const float4 ent = t[el * V + l];
          const int s0 = __float_as_int(ent.x);
          if (s0 != kInactive) gather_taps<J>(g + (ptrdiff_t)s0 * fpass, fpass, ent, acc[vp]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  // x[f][voxel - x_v0] = acc / A (das.cpp:327-328).
  const float inv = (float)(1.0 / p.A);
#pragma unroll
  for (int vp = 0; vp < VPW; ++vp) {
    const int l = (warp * VPW + vp) * 2 + half;
    int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
    int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    if (i < p.nx && j < p.ny && k < L.kend) {
      const long long flat =
          (long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * k) - L.x_v0;
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        int f = L.pass * fpass + 16 * jj + l16;
        if (f < p.F)
          x[(size_t)f * (size_t)L.x_n + (size_t)flat] =
              make_float2(acc[vp][jj].x * inv, acc[vp][jj].y * inv);
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
