// das.cu -- 3D plane-wave delay-and-sum with coherent angle compounding.
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
// B200 design: the delay of a (voxel, element, angle)
// triple does not depend on the frame, so the kernel is frames-innermost.
// One CTA owns a voxel tile and 16*J frames of one pass.  Per stage (angle a,
// block of 8 elements):
//   A  receive range r/c per (voxel, element) in FP64, with the f-number mask
//      (once per element block, reused by all angles);
//   B  per (voxel, element): tap index s0, frac and the carrier rotation in
//      FP64 -> a 16-byte table entry in shared memory; the min/max tap of each
//      element defines its time window;
//   C  one thread issues 1-D TMA bulk copies (cp.async.bulk) of each element's
//      window rows -- contiguous because frames are innermost in the IQ layout
//      -- into shared memory, completing on an mbarrier;
//   D  lanes = 16 frames x 2 voxels: each lane gathers its frames' two taps
//      from shared memory (conflict-free 128 B half-warp rows), interpolates,
//      rotates and accumulates in registers (acc[VPW][J] complex f32).
// FP64 delay math is amortised over all frames of the pass; the gather is
// served from shared memory, so HBM sees each IQ row once per tile-wave
// (L2-resident between neighbouring tiles, which run concurrently).
#include <cuda_runtime.h>

#include "common.cuh"

namespace fqfg {

constexpr int kEB = 8;  // elements per stage
constexpr int kInactive = (int)0x80000000;

FQFG_DEVICE void mbar_init(uint64_t* bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

FQFG_DEVICE void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}

// try_wait with a suspend-time hint: the waiting warp sleeps (up to `ns`)
// instead of re-issuing the probe, leaving issue slots to working warps.
FQFG_DEVICE void mbar_wait_hint(uint64_t* bar, unsigned phase, unsigned ns) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITH_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase), "r"(ns)
      : "memory");
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

FQFG_DEVICE void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
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
  int TX, TY, TZ;      // voxel tile
  int tiles_x, tiles_y;
  int kbeg, kend;      // z-slab
  int pass;
  int rcap;            // window rows that fit in shared memory
  int debug;           // 1: das2 consumers skip the gather (producer-bound timing)
  int pairy;           // das2 mode 0: the two half-warps take y-adjacent voxels (TY even)
  unsigned hint;       // das2: mbarrier try_wait suspend-time hint (ns), 0 = none
  int pf;              // das2: L2 prefetch distance in stages (0 = off)
  int exactwin;        // das2 mode 0: exact per-element windows (min/max tap index from the
                       // table; TMA issued after the table) instead of tile-box bounds
};

template <int J, int VPW, int NWARP>
__global__ void __launch_bounds__(NWARP * 32, 1)
    das_kernel(const DasParams p, const DasLaunch L, const float2* __restrict__ iq,
               float2* __restrict__ x, unsigned long long* __restrict__ counters) {
  constexpr int V = NWARP * VPW * 2;
  constexpr int NT = NWARP * 32;
  static_assert(V % 32 == 0, "a warp must not straddle two elements in phase B");
  const int fpass = 16 * J;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* win = reinterpret_cast<float2*>(smem_raw);  // [rcap][fpass]
  unsigned char* sp = smem_raw + (size_t)L.rcap * fpass * sizeof(float2);
  float4* tab = reinterpret_cast<float4*>(sp);           // [kEB][V]
  double* rc = reinterpret_cast<double*>(tab + V * kEB);  // [kEB][V]
  double* vox = rc + V * kEB;                            // [V][3]
  double* ttx = vox + 3 * V;                             // [V]
  int* wmin = reinterpret_cast<int*>(ttx + V);           // [kEB]
  int* wmax = wmin + kEB;                                // [kEB]
  int* wbase = wmax + kEB;                               // [kEB]
  int* grp = wbase + kEB;                                // [2]: group end, rows
  uint64_t* bar = reinterpret_cast<uint64_t*>(grp + 4);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, l16 = lane & 15;

  // Tile origin.
  int tile = blockIdx.x;
  const int tx = tile % L.tiles_x;
  tile /= L.tiles_x;
  const int ty = tile % L.tiles_y;
  const int tz = tile / L.tiles_y;
  const int i0 = tx * L.TX, j0 = ty * L.TY, k0 = L.kbeg + tz * L.TZ;

  for (int l = tid; l < V; l += NT) {
    int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
    int i = i0 + lx, j = j0 + ly, k = k0 + lz;
    bool ok = i < p.nx && j < p.ny && k < L.kend;
    // GridSpec::point (das.hpp:28-32): origin + index * spacing.
    vox[3 * l] = ok ? grid_coord(p.ox, i, p.sx) : __longlong_as_double(0x7ff8000000000000ll);
    vox[3 * l + 1] = grid_coord(p.oy, j, p.sy);
    vox[3 * l + 2] = grid_coord(p.oz, k, p.sz);
  }
  if (tid == 0) mbar_init(bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  float2 acc[VPW][J];
#pragma unroll
  for (int v = 0; v < VPW; ++v)
#pragma unroll
    for (int j = 0; j < J; ++j) acc[v][j] = make_float2(0.f, 0.f);

  unsigned long long n_oow = 0, n_taps = 0;
  unsigned phase = 0;
  const int nblk = (p.E + kEB - 1) / kEB;

  for (int eb = 0; eb < nblk; ++eb) {
    // ---- A: receive delay r/c and the f-number mask (das.cpp:165-170).
    int any = 0;
    for (int idx = tid; idx < V * kEB; idx += NT) {
      int l = idx % V, el = idx / V, e = eb * kEB + el;
      double v = -1.0;
      double px = vox[3 * l], py = vox[3 * l + 1], pz = vox[3 * l + 2];
      if (e < p.E && px == px) {
        double ex = __ldg(p.elem + 3 * e), ey = __ldg(p.elem + 3 * e + 1),
               ez = __ldg(p.elem + 3 * e + 2);
        bool in = !(p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum));
        if (in) {
          v = rx_delay(px, py, pz, ex, ey, ez, p.c);
          any = 1;
        }
      }
      rc[idx] = v;
    }
    if (!__syncthreads_or(any)) continue;

    for (int a = 0; a < p.A; ++a) {
      const AngleConst ac = p.ang[a];
      // ---- B0: plane-wave transmit delay per voxel (das.cpp:162).
      for (int l = tid; l < V; l += NT)
        ttx[l] = tx_delay(vox[3 * l], vox[3 * l + 2], ac.sina, ac.cosa, ac.ref, p.c);
      if (tid < kEB) {
        wmin[tid] = 0x7fffffff;
        wmax[tid] = kInactive;
      }
      __syncthreads();
      // ---- B: taps, weights and carrier rotation (das.cpp:169-197).
      // Lanes walk voxels of one element (V is a multiple of 32), so the
      // window min/max reduce in-warp before one shared atomic per warp.
      for (int idx = tid; idx < V * kEB; idx += NT) {
        int l = idx % V, el = idx / V;
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
            // exp(+i 2 pi f_c tau) via the fractional cycle count: FP64
            // reduction, then an f32 sincospi on |x| <= 1.
            double cyc = p.fc * tau;
            cyc -= rint(cyc);
            float sn, cs;
            sincospif(2.0f * (float)cyc, &sn, &cs);
            ent = make_float4(__int_as_float(s0), frac, cs, sn);
          }
        }
        const int s0v = __float_as_int(ent.x);
        const int mn = __reduce_min_sync(0xffffffffu, s0v == kInactive ? 0x7fffffff : s0v);
        const int mx = __reduce_max_sync(0xffffffffu, s0v);
        if (lane == 0) {
          if (mn != 0x7fffffff) atomicMin(&wmin[el], mn);
          if (mx != kInactive) atomicMax(&wmax[el], mx);
        }
        tab[idx] = ent;
      }
      __syncthreads();

      // ---- C/D: copy element windows (grouped to fit rcap rows), gather.
      int e_begin = 0;
      while (e_begin < kEB) {
        if (tid == 0) {
          int rows = 0, e = e_begin;
          for (; e < kEB; ++e) {
            int n = wmax[e] >= wmin[e] ? wmax[e] - wmin[e] + 2 : 0;
            if (n > L.rcap) {  // window too tall to stage: gather from global
              wbase[e] = -1;
              continue;
            }
            if (rows + n > L.rcap) break;
            wbase[e] = rows;
            rows += n;
          }
          grp[0] = e;
          grp[1] = rows;
          if (rows > 0) {
            mbar_expect_tx(bar, (unsigned)rows * fpass * sizeof(float2));
            for (int q = e_begin; q < e; ++q) {
              int n = wmax[q] >= wmin[q] ? wmax[q] - wmin[q] + 2 : 0;
              if (n == 0 || wbase[q] < 0) continue;
              size_t row0 = iq_row_index(p, a, eb * kEB + q, wmin[q] + 1);
              bulk_g2s(win + (size_t)wbase[q] * fpass, iq + row0 * fpass,
                       (unsigned)n * fpass * sizeof(float2), bar);
            }
          }
        }
        __syncthreads();
        const int e_end = grp[0];
        if (grp[1] > 0) {
          mbar_wait(bar, phase);
          phase ^= 1;
        }
        for (int el = e_begin; el < e_end; ++el) {
          if (wmax[el] < wmin[el]) continue;
          if (wbase[el] >= 0) {
            const int row_off = wbase[el] - wmin[el];
#pragma unroll
            for (int vp = 0; vp < VPW; ++vp) {
              const int l = (warp * VPW + vp) * 2 + half;
              const float4 ent = tab[el * V + l];
              const int s0 = __float_as_int(ent.x);
              if (s0 != kInactive)
                gather_taps<J>(win + (size_t)(row_off + s0) * fpass + l16, fpass, ent, acc[vp]);
            }
          } else {
            const float2* g = iq + (iq_row_index(p, a, eb * kEB + el, 0) + 1) * fpass + l16;
#pragma unroll
            for (int vp = 0; vp < VPW; ++vp) {
              const int l = (warp * VPW + vp) * 2 + half;
              const float4 ent = tab[el * V + l];
              const int s0 = __float_as_int(ent.x);
              if (s0 != kInactive) gather_taps<J>(g + (ptrdiff_t)s0 * fpass, fpass, ent, acc[vp]);
            }
          }
        }
        __syncthreads();
        e_begin = e_end;
      }
    }
  }

  // ---- output: x[f][voxel] = acc / A (das.cpp:327-328).
  const float inv = (float)(1.0 / p.A);
  const size_t N = (size_t)p.nx * p.ny * p.nz;
#pragma unroll
  for (int vp = 0; vp < VPW; ++vp) {
    const int l = (warp * VPW + vp) * 2 + half;
    int lx = l % L.TX, ly = (l / L.TX) % L.TY, lz = l / (L.TX * L.TY);
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
}

// Shared-memory bytes besides the window buffer.
template <int V>
constexpr size_t das_aux_smem() {
  return (size_t)V * kEB * 16 + (size_t)V * kEB * 8 + (size_t)V * 3 * 8 + (size_t)V * 8 +
         4 * kEB * 4 + 16 + 16;
}

}  // namespace fqfg
