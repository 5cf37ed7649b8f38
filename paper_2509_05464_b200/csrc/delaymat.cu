// delaymat.cu -- the reference's explicit sparse delay-matrix API on the GPU:
// build_delay_matrix (das.cpp:126-208) and apply_delay_matrix (das.cpp:210-222).
//
// The production DAS (das2.cu) never materialises these matrices; this file
// exists so the drop-in library still provides the reference's full
// beamforming API (its tests and any caller that inspects the operator).
// Two passes: count taps per voxel (row lengths, out-of-window pairs, the
// deepest tap for padded_samples), then fill each row in element order with
// value = weight * exp(+i 2 pi f_c tau).  All delay arithmetic is the same
// non-contracted FP64 sequence as das2's producers, so column indices are
// bit-identical to the reference; the SpMV runs in FP64 in entry order.
#include "common.cuh"

namespace fqfg {

struct DmParams {
  double sina, cosa, ref, t0, fs, c, omega, fnum;
  int E, T, interp;
  const double* elem;  // [E][3]
};

// Per voxel: taps (row length), out_of_window pairs, deepest tap index.
__global__ void dm_count_kernel(const DmParams q, const double* __restrict__ vox, size_t n,
                                unsigned long long* __restrict__ row_len,
                                unsigned long long* __restrict__ oow,
                                long long* __restrict__ last_tap) {
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c_oow = 0;
  long long last = -1;
  if (v < n) {
    double px = vox[3 * v], py = vox[3 * v + 1], pz = vox[3 * v + 2];
    double ttx = tx_delay(px, pz, q.sina, q.cosa, q.ref, q.c);
    unsigned long long len = 0;
    for (int e = 0; e < q.E; ++e) {
      double ex = q.elem[3 * e], ey = q.elem[3 * e + 1], ez = q.elem[3 * e + 2];
      if (q.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, q.fnum)) continue;
      double tau = xadd(ttx, rx_delay(px, py, pz, ex, ey, ez, q.c));
      double s = xmul(xsub(tau, q.t0), q.fs);
      bool live = false;
      if (q.interp == 0) {
        double i = round(s);
        last = max(last, (long long)fmax(fmin(i, 9.0e18), -1.0));
        if (i >= 0.0 && i < q.T) {
          ++len;
          live = true;
        }
      } else {
        double sfl = floor(s), fr = xsub(s, sfl);
        double top = xadd(sfl, fr > 0.0 ? 1.0 : 0.0);
        last = max(last, (long long)fmax(fmin(top, 9.0e18), -1.0));
        if (sfl >= 0.0 && sfl < q.T) {
          ++len;
          live = true;
        }
        double snd = xadd(sfl, 1.0);
        if (fr > 0.0 && snd >= 0.0 && snd < q.T) {
          ++len;
          live = true;
        }
      }
      c_oow += !live;
    }
    row_len[v] = len;
  }
  for (int o = 16; o > 0; o >>= 1) {
    c_oow += __shfl_xor_sync(0xffffffffu, c_oow, o);
    last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(oow, c_oow);
    atomicMax(last_tap, last);
  }
}

// Fill row v at row_ptr[v]: columns t * E + e, values weight * rot (FP64).
__global__ void dm_fill_kernel(const DmParams q, const double* __restrict__ vox, size_t n,
                               const unsigned long long* __restrict__ row_ptr,
                               int* __restrict__ col, double2* __restrict__ val) {
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double px = vox[3 * v], py = vox[3 * v + 1], pz = vox[3 * v + 2];
  double ttx = tx_delay(px, pz, q.sina, q.cosa, q.ref, q.c);
  unsigned long long at = row_ptr[v];
  for (int e = 0; e < q.E; ++e) {
    double ex = q.elem[3 * e], ey = q.elem[3 * e + 1], ez = q.elem[3 * e + 2];
    if (q.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, q.fnum)) continue;
    double tau = xadd(ttx, rx_delay(px, py, pz, ex, ey, ez, q.c));
    double s = xmul(xsub(tau, q.t0), q.fs);
    double ph = xmul(q.omega, tau);
    double rr = cos(ph), ri = sin(ph);
    if (q.interp == 0) {
      double i = round(s);
      if (i >= 0.0 && i < q.T) {
        col[at] = (int)i * q.E + e;
        val[at++] = make_double2(rr, ri);
      }
    } else {
      double sfl = floor(s), fr = xsub(s, sfl);
      if (sfl >= 0.0 && sfl < q.T) {
        double w = xsub(1.0, fr);
        col[at] = (int)sfl * q.E + e;
        val[at++] = make_double2(xmul(w, rr), xmul(w, ri));
      }
      double snd = xadd(sfl, 1.0);
      if (fr > 0.0 && snd >= 0.0 && snd < q.T) {
        col[at] = (int)snd * q.E + e;
        val[at++] = make_double2(xmul(fr, rr), xmul(fr, ri));
      }
    }
  }
}

// y[r] = sum over the row's entries (in order) of value * iq[col] (FP64,
// non-contracted complex multiply-add, as apply_delay_matrix evaluates it).
__global__ void dm_apply_kernel(size_t rows, const unsigned long long* __restrict__ row_ptr,
                                const int* __restrict__ col, const double2* __restrict__ val,
                                const double2* __restrict__ iq, double2* __restrict__ out) {
  size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double ar = 0.0, ai = 0.0;
  for (unsigned long long i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
    double2 a = val[i], b = iq[col[i]];
    ar = xadd(ar, xsub(xmul(a.x, b.x), xmul(a.y, b.y)));
    ai = xadd(ai, xadd(xmul(a.x, b.y), xmul(a.y, b.x)));
  }
  out[r] = make_double2(ar, ai);
}

}  // namespace fqfg
