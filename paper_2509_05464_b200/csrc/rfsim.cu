// rfsim.cu -- RF channel-data synthesis on the GPU: the
// reference's frequency-domain point-scatterer simulator (proj/src/rf/
// simulate.cpp, run_engine:407-503), FP64.
//
// Model (per transmit event, bins j of the pulse passband, sub-elements i):
//   path(s, i, j) = e^{i k_j r} / r * sinc(k_j g) * elev(k_j) * e^{-beta f_j r}
//   RX(s, e, j)   = sum over the element's sub-elements of path
//   TX(s, j)      = sum_e apod_e e^{i w_j tau_e} RX(s, e, j)
//   S(j, e)       = sum_s refl_s TX(s, j) RX(s, e, j)
//   rf[m][e]      = c2r( conj(S(j, e)) * pulse(j) / T )
// Engine conventions kept: passband and 40 dB cutoff, bins walked in 64-bin
// bands, the elevation factor exact at knots 8 bins apart and linear between
// them (the model's own approximation), the same expression order per bin.
// Differences (documented, ~1e-13 relative): phasors are seeded exactly at
// every 8-bin segment instead of every 64-bin band, sums over elements and
// scatter chunks are trees in a fixed order, and the inverse transform is a
// direct DFT with an exact twiddle table instead of FFTW.
//
//   rfs_tx_kernel        CTA = (8-bin segment, scatterer chunk), threads over
//                        elements: TX(s, j) for the segment's bins by a block
//                        reduction per scatterer.
//   rfs_spec_kernel      CTA = (segment, 256 elements, scatterer chunk):
//                        refl TX RX accumulated in registers over the chunk.
//   rfs_reduce_kernel    fixed-order sum of the chunk partials.
//   rfs_idft_kernel      pulse weight, conjugate, inverse DFT -> rf [T][E].
#include "common.cuh"

namespace fqfg {

constexpr int kRfsThreads = 256;
constexpr int kRfsSeg = 8;  // bins per knot segment

struct RfsParams {
  int E, v;
  double hw;           // element half width b
  double c, df;
  double beta;         // attenuation * df (the engine's cfg.beta), nepers / m per bin
  int elev;
  double wa, inv_focus, core_w, tail_w;
  int j_lo, n_bins;
  int n_seg;
};

struct RfsSeg {
  int jb0, nb, sb0, sb1;  // band start bin, band length, segment [sb0, sb1) within the band
};

FQFG_DEVICE double rfs_elev(double ysq, double e1, double e2, double k, const RfsParams& p) {
  double w2 = e1 + e2 / (k * k);
  double core = exp(-ysq / w2);
  return p.core_w * core + p.tail_w * sqrt(sqrt(core));
}

// The element's receive sums rx[jj] over its v sub-elements for the segment's
// bins (accumulate_band:284-330 arithmetic, segment-seeded).
FQFG_DEVICE void rfs_rx(const RfsParams& p, const RfsSeg& sg, double px, double py, double pz,
                        double ex, double ey, double ez, double (&rr)[kRfsSeg],
                        double (&ri)[kRfsSeg]) {
  constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
  const double dk = kTwoPi * p.df / p.c;
  const int js = sg.jb0 + sg.sb0;
  const double fs_ = js * p.df;
  const double ks = kTwoPi * fs_ / p.c;
  const double att_k = p.beta * fs_ / p.df;
  const int hi = sg.sb1 < sg.nb ? sg.sb1 : sg.nb - 1;
  const double k_a = kTwoPi * (sg.jb0 + sg.sb0) * p.df / p.c;
  const double k_b = kTwoPi * (sg.jb0 + hi) * p.df / p.c;
  const double inv_den = hi > sg.sb0 ? 1.0 / (hi - sg.sb0) : 0.0;
  const double ysq = py * py;
#pragma unroll
  for (int q = 0; q < kRfsSeg; ++q) rr[q] = ri[q] = 0.0;
  for (int mu = 0; mu < p.v; ++mu) {
    const double off = ((mu + 0.5) / p.v - 0.5) * 2.0 * p.hw;
    const double dx = __dsub_rn(px, __dadd_rn(ex, off)), dy = __dsub_rn(py, ey),
                 dz = __dsub_rn(pz, ez);
    double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                    __dmul_rn(dz, dz)));
    r = fmax(r, 1e-6);
    const double inv_r = 1.0 / r;
    double g = fmax(fabs(__dmul_rn(__dmul_rn(p.hw, dx), inv_r)), 1e-12);
    const double inv_g = 1.0 / g;
    double st_re, st_im, ss_re, ss_im, ph_re, ph_im, sp_re, sp_im;
    sincos(dk * r, &st_im, &st_re);
    sincos(dk * g, &ss_im, &ss_re);
    sincos(ks * r, &ph_im, &ph_re);
    sincos(ks * g, &sp_im, &sp_re);
    double att = exp(-att_k * r);
    const double arat = exp(-p.beta * r);
    double d0 = 1.0, dd = 0.0;
    if (p.elev) {
      const double a = p.wa * (1.0 - r * p.inv_focus);
      const double e1 = a * a;
      const double b2 = 2.0 * r / p.wa;
      const double e2 = b2 * b2;
      d0 = rfs_elev(ysq, e1, e2, k_a, p);
      const double d1 = rfs_elev(ysq, e1, e2, k_b, p);
      dd = (d1 - d0) * inv_den;
    }
#pragma unroll
    for (int q = 0; q < kRfsSeg; ++q) {
      const int jj = sg.sb0 + q;
      if (jj < sg.sb1) {
        const double invk = p.c / (kTwoPi * (sg.jb0 + jj) * p.df);
        const double dir = __dmul_rn(__dmul_rn(sp_im, inv_g), invk);
        const double amp =
            __dmul_rn(__dmul_rn(__dmul_rn(inv_r, att), __dadd_rn(d0, __dmul_rn(dd, (double)q))),
                      dir);
        rr[q] = __dadd_rn(rr[q], __dmul_rn(amp, ph_re));
        ri[q] = __dadd_rn(ri[q], __dmul_rn(amp, ph_im));
        const double nr = __dsub_rn(__dmul_rn(ph_re, st_re), __dmul_rn(ph_im, st_im));
        ph_im = __dadd_rn(__dmul_rn(ph_re, st_im), __dmul_rn(ph_im, st_re));
        ph_re = nr;
        const double ns = __dsub_rn(__dmul_rn(sp_re, ss_re), __dmul_rn(sp_im, ss_im));
        sp_im = __dadd_rn(__dmul_rn(sp_re, ss_im), __dmul_rn(sp_im, ss_re));
        sp_re = ns;
        att = __dmul_rn(att, arat);
      }
    }
  }
}

__global__ void __launch_bounds__(kRfsThreads)
    rfs_tx_kernel(const RfsParams p, const RfsSeg* __restrict__ segs,
                  const double* __restrict__ pos, size_t n_scat, size_t chunk,
                  const double* __restrict__ elem, const double* __restrict__ delays,
                  const double* __restrict__ apod, double2* __restrict__ tx) {
  constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
  __shared__ double red[kRfsThreads / 32][2 * kRfsSeg];
  const RfsSeg sg = segs[blockIdx.x];
  const size_t s0 = (size_t)blockIdx.y * chunk, s1 = min(n_scat, s0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double fs_ = (sg.jb0 + sg.sb0) * p.df;
  for (size_t s = s0; s < s1; ++s) {
    const double px = pos[3 * s], py = pos[3 * s + 1], pz = pos[3 * s + 2];
    double tr[kRfsSeg], ti[kRfsSeg];
#pragma unroll
    for (int q = 0; q < kRfsSeg; ++q) tr[q] = ti[q] = 0.0;
    for (int e = threadIdx.x; e < p.E; e += blockDim.x) {
      double rr[kRfsSeg], ri[kRfsSeg];
      rfs_rx(p, sg, px, py, pz, elem[3 * e], elem[3 * e + 1], elem[3 * e + 2], rr, ri);
      const double tau = delays[e], w = apod[e];
      double cr, ci, sr, si;
      sincos(kTwoPi * fs_ * tau, &ci, &cr);
      sincos(kTwoPi * p.df * tau, &si, &sr);
#pragma unroll
      for (int q = 0; q < kRfsSeg; ++q) {
        tr[q] = __dadd_rn(tr[q], __dmul_rn(w, __dsub_rn(__dmul_rn(cr, rr[q]), __dmul_rn(ci, ri[q]))));
        ti[q] = __dadd_rn(ti[q], __dmul_rn(w, __dadd_rn(__dmul_rn(cr, ri[q]), __dmul_rn(ci, rr[q]))));
        const double nr = __dsub_rn(__dmul_rn(cr, sr), __dmul_rn(ci, si));
        ci = __dadd_rn(__dmul_rn(cr, si), __dmul_rn(ci, sr));
        cr = nr;
      }
    }
#pragma unroll
    for (int q = 0; q < kRfsSeg; ++q) {
      for (int o = 16; o > 0; o >>= 1) {
        tr[q] += __shfl_xor_sync(0xffffffffu, tr[q], o);
        ti[q] += __shfl_xor_sync(0xffffffffu, ti[q], o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < kRfsSeg; ++q) {
        red[warp][2 * q] = tr[q];
        red[warp][2 * q + 1] = ti[q];
      }
    }
    __syncthreads();
    if (threadIdx.x < 2 * kRfsSeg) {
      double a = 0.0;
      for (int w = 0; w < kRfsThreads / 32; ++w) a += red[w][threadIdx.x];
      const int q = threadIdx.x >> 1, jj = sg.sb0 + q;
      if (jj < sg.sb1) {
        double* t = reinterpret_cast<double*>(tx + s * (size_t)p.n_bins + (sg.jb0 - p.j_lo + jj));
        t[threadIdx.x & 1] = a;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kRfsThreads)
    rfs_spec_kernel(const RfsParams p, const RfsSeg* __restrict__ segs,
                    const double* __restrict__ pos, const double* __restrict__ refl,
                    size_t n_scat, size_t chunk, const double* __restrict__ elem,
                    const double2* __restrict__ tx, double2* __restrict__ part) {
  const RfsSeg sg = segs[blockIdx.x];
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  const size_t s0 = (size_t)blockIdx.z * chunk, s1 = min(n_scat, s0 + chunk);
  if (e >= p.E) return;
  const double ex = elem[3 * e], ey = elem[3 * e + 1], ez = elem[3 * e + 2];
  double ar[kRfsSeg], ai[kRfsSeg];
#pragma unroll
  for (int q = 0; q < kRfsSeg; ++q) ar[q] = ai[q] = 0.0;
  const int jrow = sg.jb0 - p.j_lo + sg.sb0;
  for (size_t s = s0; s < s1; ++s) {
    double rr[kRfsSeg], ri[kRfsSeg];
    rfs_rx(p, sg, pos[3 * s], pos[3 * s + 1], pos[3 * s + 2], ex, ey, ez, rr, ri);
    const double rs = refl[s];
#pragma unroll
    for (int q = 0; q < kRfsSeg; ++q) {
      if (sg.sb0 + q < sg.sb1) {
        const double2 t = tx[s * (size_t)p.n_bins + jrow + q];
        const double cr = __dmul_rn(rs, t.x), ci = __dmul_rn(rs, t.y);
        ar[q] = __dadd_rn(ar[q], __dsub_rn(__dmul_rn(cr, rr[q]), __dmul_rn(ci, ri[q])));
        ai[q] = __dadd_rn(ai[q], __dadd_rn(__dmul_rn(cr, ri[q]), __dmul_rn(ci, rr[q])));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kRfsSeg; ++q)
    if (sg.sb0 + q < sg.sb1)
      part[((size_t)blockIdx.z * p.n_bins + jrow + q) * p.E + e] = make_double2(ar[q], ai[q]);
}

__global__ void rfs_reduce_kernel(const double2* __restrict__ part, int n_chunk, size_t n,
                                  double2* __restrict__ spec) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = part[i];
  for (int c = 1; c < n_chunk; ++c) {
    const double2 b = part[(size_t)c * n + i];
    a.x += b.x;
    a.y += b.y;
  }
  spec[i] = a;
}

// rf[m][e] = sum_j 2 Re( conj(S(j, e)) w_j e^{2 pi i j m / T} ) (the c2r
// transform of bins j_lo..j_hi, run_engine:478-503); twiddles from an exact
// table indexed by (j m) mod T.
__global__ void rfs_idft_kernel(const double2* __restrict__ spec, const double* __restrict__ w,
                                const double2* __restrict__ twid, int T, int E, int j_lo,
                                int n_bins, double* __restrict__ out64,
                                float* __restrict__ out32) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)T * E) return;
  const int m = (int)(idx / E), e = (int)(idx % E);
  double acc = 0.0;
  for (int b = 0; b < n_bins; ++b) {
    const int j = j_lo + b;
    const double2 s = spec[(size_t)b * E + e];
    const double in_re = s.x * w[b], in_im = -s.y * w[b];
    const double2 t = twid[((long long)j * m) % T];
    acc += 2.0 * (in_re * t.x - in_im * t.y);
  }
  if (out64) out64[idx] = acc;
  if (out32) out32[idx] = (float)acc;
}

}  // namespace fqfg
