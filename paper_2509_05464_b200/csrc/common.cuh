// common.cuh -- shared device helpers and launch parameter structs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define FQFG_DEVICE __device__ __forceinline__

namespace fqfg {

constexpr double kPi = 3.14159265358979323846;

// ---- DAS ---------------------------------------------------------------------

constexpr int kMaxAngles = 64;

// Per-angle constants of one plane-wave transmit (das.cpp:143-145).
struct AngleConst {
  double sina, cosa, ref;  // ref = min_n x_n sin(a)
  double t0;
};

// Everything the demod and DAS kernels need about one ensemble.  Passed by
// value (kernel parameter space), so it stays < 4 KB.
struct DasParams {
  int nx, ny, nz;
  double ox, oy, oz, sx, sy, sz;  // grid origin / spacing
  int E, A, T, F;
  int fpass;      // frames per pass (16 * J)
  int npass;      // ceil(F / fpass)
  double fs, c, fc, fnum;
  int interp;     // 1 linear, 0 nearest
  int taps;       // FIR taps
  int iq_row0;    // first IQ row held per (angle, element) in the pass buffer
  int iq_rows;    // rows held (T + 2 for the whole record; a slab's readable rows)
  const double* elem;  // [E][3]
  AngleConst ang[kMaxAngles];
};

// ---- packed FP32 pairs (FFMA2 on sm_100): a float2 held in one 64-bit register
FQFG_DEVICE unsigned long long f2pk(uint32_t lo, uint32_t hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
FQFG_DEVICE unsigned long long f2bc(float a) { return f2pk(__float_as_uint(a), __float_as_uint(a)); }
FQFG_DEVICE unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                     unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// ---- reference-exact FP64 geometry ------------------------------------------
// The reference is built without FMA (proj/CMakeLists.txt:9, baseline
// x86-64), so every delay is a sequence of separately rounded IEEE ops.  The
// _rn intrinsics are never contracted, which makes the tap index, the
// interpolation weight and the aperture decision bit-identical to
// build_delay_matrix (das.cpp:159-197) for identical inputs.
FQFG_DEVICE double xmul(double a, double b) { return __dmul_rn(a, b); }
FQFG_DEVICE double xadd(double a, double b) { return __dadd_rn(a, b); }
FQFG_DEVICE double xsub(double a, double b) { return __dsub_rn(a, b); }

// glibc 2.35+ hypot (the non-FMA kernel the reference's std::hypot resolves
// to), restated; bit-identical to glibc on 2e7 random pairs
// (tests/test_host.py::test_hypot_restatement_matches_glibc).  Valid for the
// normal range |x|, |y| in [2^-500, 2^500] that probe geometry occupies.
FQFG_DEVICE double ref_hypot(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (ay > ax) {
    double t = ax;
    ax = ay;
    ay = t;
  }
  if (ay == 0.0) return ax;
  double h = __dsqrt_rn(xadd(xmul(ax, ax), xmul(ay, ay)));
  double t1, t2;
  if (h <= xmul(2.0, ay)) {
    double delta = xsub(h, ay);
    t1 = xmul(ax, xsub(xmul(2.0, delta), ax));
    t2 = xmul(xsub(delta, xmul(2.0, xsub(ax, ay))), delta);
  } else {
    double delta = xsub(h, ax);
    t1 = xmul(xmul(2.0, delta), xsub(ax, xmul(2.0, ay)));
    t2 = xadd(xmul(xsub(xmul(4.0, delta), ay), ay), xmul(delta, delta));
  }
  return xsub(h, __ddiv_rn(xadd(t1, t2), xmul(2.0, h)));
}

// GridSpec::point (das.hpp:28-32): origin + index * spacing.
FQFG_DEVICE double grid_coord(double o, int i, double s) { return xadd(o, xmul((double)i, s)); }

// f-number cut (das.cpp:165-168): true when the element is OUTSIDE.
FQFG_DEVICE bool outside_aperture(double px, double py, double pz, double ex, double ey,
                                  double ez, double fnum) {
  double lat = ref_hypot(xsub(px, ex), xsub(py, ey));
  return xmul(xmul(lat, 2.0), fnum) > xsub(pz, ez);
}

// |p - e| / c (das.cpp:169-170; Vec3 norm = sqrt(x*x + y*y + z*z)).
FQFG_DEVICE double rx_delay(double px, double py, double pz, double ex, double ey, double ez,
                            double c) {
  double dx = xsub(px, ex), dy = xsub(py, ey), dz = xsub(pz, ez);
  double r = __dsqrt_rn(xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz)));
  return __ddiv_rn(r, c);
}

// (p.x sin a + p.z cos a - ref) / c (das.cpp:162).
FQFG_DEVICE double tx_delay(double px, double pz, double sina, double cosa, double ref, double c) {
  return __ddiv_rn(xsub(xadd(xmul(px, sina), xmul(pz, cosa)), ref), c);
}

// IQ of one frame pass, layout [angle][element][row][frame-in-pass] complex64.
// Row r holds sample t = r - 1; rows 0 and T + 1 are zero so a tap pair
// (s0, s0 + 1) with s0 in [-1, T - 1] is always addressable.  Only rows
// [iq_row0, iq_row0 + iq_rows) are stored: the rows some voxel of the launch's
// slab can read (slab_rows), never a tap outside them.
FQFG_DEVICE long long iq_row_index(const DasParams& p, int a, int e, int row) {
  return ((long long)a * p.E + e) * (long long)p.iq_rows + (row - p.iq_row0);
}

}  // namespace fqfg
