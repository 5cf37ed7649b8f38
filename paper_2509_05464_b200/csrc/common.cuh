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
  const double* elem;  // [E][3]
  AngleConst ang[kMaxAngles];
};

// IQ of one frame pass, layout [angle][element][row][frame-in-pass] complex64.
// Row r holds sample t = r - 1; rows 0 and T + 1 are zero so a tap pair
// (s0, s0 + 1) with s0 in [-1, T - 1] is always addressable.
FQFG_DEVICE size_t iq_row_index(const DasParams& p, int a, int e, int row) {
  return ((size_t)a * p.E + e) * (size_t)(p.T + 2) + row;
}

}  // namespace fqfg
