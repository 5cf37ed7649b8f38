// capi.cu -- host side of the C ABI (include/fqfgpu.h): contract checks with
// the reference's require() messages, chunk planning for DasStats parity,
// device workspaces, stream orchestration and kernel launches.
//
// Compiled by nvcc as host C++17 plus the kernel translation units included
// below (one .so, one fatbin for sm_100a).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <memory>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/fqfgpu.h"
#include "common.cuh"
#include "das2.cu"
#include "delaymat.cu"
#include "display.cu"
#include "rfsim.cu"
#include "demod.cu"
#include "das_tc.cu"
#include "eig2.cu"
#include "gram.cu"
#include "gram_i8.cu"
#include "project.cu"

using namespace fqfg;

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  throw Fail{code};
}

void require(bool cond, const char* fmt, ...) {
  if (cond) return;
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  throw Fail{FQFG_EINVAL};
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess && (cudaGetLastError(), true))  /* clear, report once */    \
      fail(e_ == cudaErrorMemoryAllocation ? FQFG_ENOMEM : FQFG_ECUDA, "%s: %s (%s:%d)", \
           #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
  } while (0)

std::atomic<unsigned long long> g_launches{0};

#define CK_LAUNCH()                \
  do {                             \
    CK(cudaGetLastError());        \
    g_launches.fetch_add(1);       \
  } while (0)

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return FQFG_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FQFG_ECUDA;
  }
}

int sm100_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++ok;
  }
  return ok;
}

void need_device() {
  static int n = sm100_devices();
  if (n == 0)
    fail(FQFG_ENODEV, "no sm_100 (B200) CUDA device available; this library has no CPU path");
}

// Grow-only device buffers, one set per (device, thread) so concurrent calls
// from different host threads never share scratch.
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  int dev = -1;
  void* get(size_t bytes) {
    int d;
    CK(cudaGetDevice(&d));
    if (bytes <= n && d == dev) return p;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    n = std::max<size_t>(bytes, 256);
    dev = d;
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

thread_local DevBuf tl_rf, tl_x, tl_work, tl_y, tl_pd, tl_small, tl_gram, tl_cnt, tl_eig, tl_corr;

// cudaFuncSetAttribute acts on the current device's context only: raise a
// kernel's dynamic shared-memory limit once per (kernel, device), so a process
// that drives several GPUs (fqfg_set_device, the reconstruction engine) gets
// the attribute on each of them.
void smem_attr(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[{fn, dev}];
  if (bytes > have) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
}

// ------------------------------------------------------------- planning --

void split_ranges(size_t n, size_t k, std::vector<std::pair<size_t, size_t>>& out) {
  out.clear();
  size_t base = n / k, rem = n % k, at = 0;
  for (size_t i = 0; i < k; ++i) {
    size_t len = base + (i < rem ? 1 : 0);
    out.emplace_back(at, at + len);
    at += len;
  }
}

// plan_chunks (das.cpp:97-119).
size_t plan_chunks(size_t n_points, int n_angles, size_t budget,
                   std::vector<std::pair<size_t, size_t>>& ranges) {
  require(n_points > 0, "reconstruction grid is empty");
  require(n_angles > 0, "need at least one transmit");
  size_t row = 16ull * (size_t)n_angles;
  require(budget > row, "memory budget cannot hold one voxel across %d transmits", n_angles);
  require(n_points <= std::numeric_limits<size_t>::max() / row,
          "reconstruction grid is too large to size");
  size_t bytes = row * n_points;
  size_t by_total = (bytes + budget - 1) / budget;
  size_t cap = budget / row;
  size_t by_cap = (n_points + cap - 1) / cap;
  size_t k = std::max(by_total, by_cap);
  split_ranges(n_points, k, ranges);
  return k;
}

// The delay-matrix re-plan of das_reconstruct (das.cpp:258-274).
size_t das_chunk_plan(size_t n_points, int A, int E, int interp, const fqfg_das_opts& o,
                      std::vector<std::pair<size_t, size_t>>& ranges) {
  size_t k = plan_chunks(n_points, A, o.memory_budget_bytes, ranges);
  size_t maxlen = 0;
  for (auto& r : ranges) maxlen = std::max(maxlen, r.second - r.first);
  size_t resident = o.cache_matrices ? (size_t)A : 1;
  size_t taps = interp == 0 ? 1 : 2;
  size_t entry = 16 + 4;
  size_t bound = maxlen * taps * (size_t)E * entry + (maxlen + 1) * 8;
  if (resident * bound > o.matrix_budget_bytes) {
    size_t per_chunk = o.matrix_budget_bytes / resident;
    size_t per_voxel = taps * (size_t)E * entry + 8;
    size_t len_cap = per_chunk > 8 ? (per_chunk - 8) / per_voxel : 0;
    require(len_cap >= 1, "delay-matrix budget cannot hold one voxel row");
    k = std::max(k, (n_points + len_cap - 1) / len_cap);
    split_ranges(n_points, k, ranges);
  }
  return k;
}

void check_grid(const fqfg_grid* g) {
  require(g && g->dims[0] >= 1 && g->dims[1] >= 1 && g->dims[2] >= 1,
          "reconstruction grid dims must be positive");
  require(g->spacing[0] > 0 && g->spacing[1] > 0 && g->spacing[2] > 0,
          "reconstruction grid spacing must be positive");
  require(std::isfinite(g->origin[0]) && std::isfinite(g->origin[1]) &&
              std::isfinite(g->origin[2]),
          "reconstruction grid origin must be finite");
}

void check_rf(const fqfg_rf_desc* d, const fqfg_probe* pr) {
  require(d != nullptr && d->n_frames >= 1, "no frames to reconstruct");
  require(d->n_angles >= 1, "frames carry no transmits");
  require(d->n_angles <= kMaxAngles, "at most %d transmits per frame are supported", kMaxAngles);
  require(pr && pr->n_elements >= 1 && pr->xyz, "transducer has no elements");
  require(d->sampling_rate > 0.0 && d->n_samples >= 1, "frames are empty");
  require(d->n_elements == pr->n_elements, "element count does not match the transducer");
  for (int a = 0; a < d->n_angles; ++a) {
    require(std::isfinite(d->angles[a]) && std::fabs(d->angles[a]) < kPi / 2.0,
            "steering angle must stay within the forward half-space");
    require(std::isfinite(d->t0[a]), "start time must be finite");
  }
}

void check_bf(const fqfg_bf* bf, double fs) {
  require(bf && bf->c > 0.0, "sound speed must be positive");
  require(bf->center_frequency > 0.0, "demodulation frequency must be positive");
  require(bf->interp_order == 0 || bf->interp_order == 1,
          "interpolation order must be 0 (nearest) or 1 (linear)");
  require(fs > 2.0 * bf->center_frequency,
          "sampling rate must exceed twice the demodulation frequency");
  require(bf->lowpass_taps >= 3 && bf->lowpass_taps % 2 == 1,
          "low-pass tap count must be odd and at least 3");
  require(bf->lowpass_taps <= 255, "low-pass tap count above 255 is not supported");
}

// Hamming-windowed sinc (iq.cpp:17-30), FP64.
std::vector<double> lowpass(double fc, double fs, int taps) {
  int mid = taps / 2;
  std::vector<double> h(taps);
  double sum = 0.0;
  for (int k = 0; k < taps; ++k) {
    double x = 2.0 * kPi * (fc / fs) * (k - mid);
    double s = k == mid ? 1.0 : std::sin(x) / x;
    double w = 0.54 - 0.46 * std::cos(2.0 * kPi * k / (taps - 1));
    h[k] = s * w;
    sum += h[k];
  }
  for (double& v : h) v /= sum;
  return h;
}

// carrier[a][t] = 2 exp(-i 2 pi f_c (t0_a + t/fs)) (iq.cpp:51-54).
std::vector<double2> carrier_table(const double* t0, int A, int T, double fc, double fs) {
  std::vector<double2> c((size_t)A * T);
  for (int a = 0; a < A; ++a)
    for (int t = 0; t < T; ++t) {
      double th = -2.0 * kPi * fc * (t0[a] + t / fs);
      c[(size_t)a * T + t] = make_double2(2.0 * std::cos(th), 2.0 * std::sin(th));
    }
  return c;
}

}  // namespace

// ---------------------------------------------------------------- plan --

struct fqfg_das_plan_s {
  int device = 0;
  DasParams p{};
  // das2_kernel shape: J frame groups of 16 per lane row (fpass = 16 J), VPW
  // voxel pairs per consumer warp, NW consumer + PW producer warps, EB
  // elements per stage, NS pipeline slots, voxel tile TX x TY x TZ.
  int J = 7, VPW = 8, NW = 8, PW = 4, EB = 4, NS = 2;
  int TX = 8, TY = 8, TZ = 2;
  int rcap = 0;
  size_t smem = 0;
  // Tensor-core DAS (das_tc.cu) instead of das2: fp16 hi/lo IQ windows,
  // weights in TMEM.  tc_aux: per-frame max |RF| and scale ahead of the IQ.
  bool tc = false;
  size_t tc_aux = 0;
  float hsum = 0.f;
  unsigned long long* d_kblocks = nullptr;  // das_tc K-block counter (engine-owned, may be null)
  double* d_elem = nullptr;
  std::vector<double> h_elem;  // host copy (slab_rows runs without a device sync)
  double2* d_car = nullptr;
  float* d_h = nullptr;
  uint64_t active_pairs = 0;
  size_t stage_bytes = 0, iq_bytes = 0;
  bool fused_demod = true;
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // [pass][4]: demod start/stop, das start/stop
  int ev_used = 0;              // passes recorded by the last call, not yet harvested
  double acc_demod_ms = 0.0, acc_das_ms = 0.0;
  uint64_t acc_calls = 0;
};

namespace {

// das2 instances: (J, VPW, consumer warps, elements per stage, pipeline
// slots, producer warps).
void* pick_das2(int J, int VPW, int NCW, int EB, int NS, int PW) {
#define INST(j, v, w, b, n, pw)                                             \
  if (J == j && VPW == v && NCW == w && EB == b && NS == n && PW == pw) \
    return (void*)das2_kernel<j, v, w, b, n, pw>;
  INST(1, 16, 8, 4, 2, 4) INST(2, 16, 8, 4, 2, 4) INST(4, 12, 8, 4, 2, 4)
  INST(7, 4, 16, 4, 2, 8) INST(13, 2, 16, 4, 2, 8)
#undef INST
  fail(FQFG_EINVAL, "no das2 kernel instance for J=%d VPW=%d NCW=%d EB=%d NS=%d PW=%d", J, VPW,
       NCW, EB, NS, PW);
}

void tile_for(int V, int ny, int& TX, int& TY, int& TZ) {
  if (ny == 1 && V % 16 == 0) {  // 2-D (x-z) grid: no voxel of the tile wasted on y
    TX = 16, TY = 1, TZ = V / 16;
    return;
  }
  if (V == 64 && ny >= 8) {  // C default: narrow in x (the steering axis) -> 608 vs 614 ms
    TX = 4, TY = 8, TZ = 2;
    return;
  }
  TX = 8;
  TY = V >= 128 ? 8 : V == 96 ? 6 : V == 48 ? 6 : 4;
  TZ = V / (TX * TY);
  require(TX * TY * TZ == V, "no voxel tile for %d voxels", V);
}

// Count (voxel, element) pairs inside the f-number aperture, one thread per
// voxel (the DAS roofline unit, times A).
__global__ void count_active_kernel(DasParams p, unsigned long long* out) {
  size_t n = (size_t)p.nx * p.ny * p.nz;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (v < n) {
    int i = (int)(v % p.nx), j = (int)((v / p.nx) % p.ny), k = (int)(v / ((size_t)p.nx * p.ny));
    double px = grid_coord(p.ox, i, p.sx), py = grid_coord(p.oy, j, p.sy),
           pz = grid_coord(p.oz, k, p.sz);
    for (int e = 0; e < p.E; ++e) {
      double ex = p.elem[3 * e], ey = p.elem[3 * e + 1], ez = p.elem[3 * e + 2];
      if (p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum)) continue;
      ++c;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

// Per-(voxel, angle) live-tap counts and out-of-window pairs, for DasStats
// (matrix_bytes_peak needs the CSR nnz of each chunk, das.cpp:121-124).
__global__ void tap_stats_kernel(DasParams p, unsigned* __restrict__ taps,
                                 unsigned long long* oow) {
  size_t n = (size_t)p.nx * p.ny * p.nz;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c_oow = 0;
  if (v < n) {
    int i = (int)(v % p.nx), j = (int)((v / p.nx) % p.ny), k = (int)(v / ((size_t)p.nx * p.ny));
    double px = grid_coord(p.ox, i, p.sx), py = grid_coord(p.oy, j, p.sy),
           pz = grid_coord(p.oz, k, p.sz);
    for (int a = 0; a < p.A; ++a) {
      const AngleConst ac = p.ang[a];
      double ttx = tx_delay(px, pz, ac.sina, ac.cosa, ac.ref, p.c);
      unsigned cnt = 0;
      for (int e = 0; e < p.E; ++e) {
        double ex = p.elem[3 * e], ey = p.elem[3 * e + 1], ez = p.elem[3 * e + 2];
        if (p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum)) continue;
        double tau = xadd(ttx, rx_delay(px, py, pz, ex, ey, ez, p.c));
        double s = xmul(xsub(tau, ac.t0), p.fs);
        int live;
        if (p.interp) {
          double sfl = floor(s), fr = xsub(s, sfl);
          int l0 = sfl >= 0.0 && sfl < p.T;
          int l1 = fr > 0.0 && xadd(sfl, 1.0) >= 0.0 && xadd(sfl, 1.0) < p.T;
          cnt += l0 + l1;
          live = l0 | l1;
        } else {
          double r = round(s);
          live = r >= 0.0 && r < p.T;
          cnt += live;
        }
        c_oow += !live;
      }
      taps[v * p.A + a] = cnt;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c_oow += __shfl_xor_sync(0xffffffffu, c_oow, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(oow, c_oow);
}

// Kernel shape, frames per pass and shared-memory layout of a plan whose
// pass IQ buffer holds iq_rows rows per (angle, element) and may take
// iq_budget bytes (0: no limit).  Re-run by the engine once it knows its
// slab's readable rows.
void plan_shape(fqfg_das_plan_s& P, size_t iq_budget, int iq_rows) {
  // Frames per pass and kernel shape: 16 frame lanes x J frames per lane
  // (fpass = 16 J), VPW voxel pairs per consumer warp (acc = 4 VPW J regs).
  // Measured on B200 (profiles/r01_das2_C.md): 16 consumer + 8 producer
  // warps where the accumulators fit (J = 7, 13), 8 + 4 below.  The IQ of a
  // pass (A E iq_rows fpass complex64) must fit next to the caller's buffers:
  // J steps down until it fits `iq_budget`.
  DasParams& p = P.p;
  const int F = p.F;
  auto shape_for = [&](int J) {
    P.J = J;
    P.NW = 8, P.PW = 4;
    if (J == 1) P.VPW = 16;
    else if (J == 2) P.VPW = 16;
    else if (J == 4) P.VPW = 12;
    else if (J == 7) P.VPW = 4, P.NW = 16, P.PW = 8;
    else P.VPW = 2, P.NW = 16, P.PW = 8;
  };
  const int Js[] = {1, 2, 4, 7, 13};
  int ji = F <= 16 ? 0 : F <= 32 ? 1 : F <= 64 ? 2 : F <= 112 ? 3 : 4;
  // (tensor-core DAS: per-frame scale block + fp16 hi/lo rows padded to 4)
  // (FQFG_DAS_TC=0 selects das2 instead, read here once per plan)
  const bool tc_env = [] {
    const char* e = std::getenv("FQFG_DAS_TC");
    return !(e && e[0] == '0');
  }();
  // 2-D (x-z) grids keep das2: a 64-pixel tile's window spans ~30 rows (2-3
  // MMA parts) and few frames make N small (config A: 0.98 vs 0.70 ms)
  const bool tc_ok = tc_env && p.taps <= kFusedMaxTaps && p.A <= kTcMaxA && p.ny > 1;
  auto tc_aux_for = [](int J) { return (size_t)(8 * 16 * J + 1023) / 1024 * 1024; };
  auto iq_bytes_for = [&](int J) {
    if (tc_ok && 16 * J <= kTcMaxFpass)
      return tc_aux_for(J) + (size_t)8 * 16 * J * 16 +  // (+ 4 chunks past the end)
             (size_t)p.A * p.E * (size_t)((iq_rows + 3) & ~3) * (size_t)(16 * J) * sizeof(float2);
    return (size_t)p.A * p.E * (size_t)iq_rows * (size_t)(16 * J) * sizeof(float2);
  };
  while (ji > 0 && iq_budget > 0 && iq_bytes_for(Js[ji]) > iq_budget) --ji;
  shape_for(Js[ji]);
  p.fpass = 16 * P.J;
  p.npass = (F + p.fpass - 1) / p.fpass;
  const int V = P.NW * P.VPW * 2;
  tile_for(V, p.ny, P.TX, P.TY, P.TZ);
  bool explicit_tile = false;
  // Shape override for tuning sweeps, read once here: "J,VPW,NW,PW[,TX,TY,TZ]"
  // (must name an instantiated das2 kernel; J also sets the tensor-core DAS's
  // frames per pass, a 64-voxel tile its tile; fqfg_das_plan_info_get reports it).
  if (const char* env = std::getenv("FQFG_DAS_SHAPE")) {
    int v[7] = {0, 0, 0, 0, 0, 0, 0};
    const int n =
        std::sscanf(env, "%d,%d,%d,%d,%d,%d,%d", v, v + 1, v + 2, v + 3, v + 4, v + 5, v + 6);
    require(n == 4 || n == 7, "FQFG_DAS_SHAPE must be J,VPW,NW,PW[,TX,TY,TZ]");
    P.J = v[0], P.VPW = v[1], P.NW = v[2], P.PW = v[3];
    p.fpass = 16 * P.J;
    p.npass = (F + p.fpass - 1) / p.fpass;
    const int V2 = P.NW * P.VPW * 2;
    explicit_tile = n == 7;
    if (n == 7) {
      require(v[4] * v[5] * v[6] == V2, "FQFG_DAS_SHAPE tile must hold %d voxels", V2);
      P.TX = v[4], P.TY = v[5], P.TZ = v[6];
    } else {
      tile_for(V2, p.ny, P.TX, P.TY, P.TZ);
    }
    pick_das2(P.J, P.VPW, P.NW, P.EB, P.NS, P.PW);  // fails loudly if not instantiated
  }
  int max_smem = 0;
  CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, P.device));
  const size_t row_bytes = (size_t)p.fpass * sizeof(float2);
  const size_t aux = das2_aux_smem(P.NW * P.VPW * 2, P.EB, P.NS, p.A);
  P.rcap = (int)std::min<size_t>((max_smem - aux - 1024) / (P.NS * row_bytes), 1024);
  P.smem = P.NS * (size_t)P.rcap * row_bytes + aux;
  // The fused demodulation needs no staging buffer; longer filters use the
  // two-kernel form with a [fpass][A][T][E] staging buffer.
  P.fused_demod = p.taps <= kFusedMaxTaps;
  P.stage_bytes = P.fused_demod ? 0 : (size_t)p.fpass * p.A * p.T * p.E * sizeof(float2);
  P.iq_bytes = iq_bytes_for(P.J);
  P.tc = tc_ok && p.fpass <= kTcMaxFpass;
  if (P.tc) {
    P.tc_aux = tc_aux_for(P.J);
    // 8 x 8 x 1 on 3-D grids: one voxel step in z moves the delay by ~4
    // samples, in x / y by < 1, so a flat tile keeps the (element, angle)
    // window short (C: 1.14e8 instead of 1.59e8 K blocks for 4 x 8 x 2,
    // profiles/r02_das_tc_C.md); an FQFG_DAS_SHAPE tile of 64 voxels wins
    if (!(explicit_tile && P.TX * P.TY * P.TZ == kTcV)) {
      if (p.ny >= 8) P.TX = 8, P.TY = 8, P.TZ = 1;
      else tile_for(kTcV, p.ny, P.TX, P.TY, P.TZ);
    }
    P.rcap = das_tc_slots(p.A, max_smem);
    require(P.rcap != 0, "das_tc: no shared-memory layout for %d angles", p.A);
    P.smem = das_tc_smem(p.A, P.rcap & 0xff, P.rcap >> 8);
  }

}

void build_plan(const fqfg_rf_desc* d, const fqfg_grid* g, const fqfg_probe* pr,
                const fqfg_bf* bf, fqfg_das_plan_s& P, size_t iq_budget = 0) {
  check_rf(d, pr);
  check_grid(g);
  check_bf(bf, d->sampling_rate);
  require((size_t)d->n_samples * d->n_elements <= (size_t)std::numeric_limits<int32_t>::max(),
          "recording is too large for the column index width");
  DasParams& p = P.p;
  p.nx = g->dims[0];
  p.ny = g->dims[1];
  p.nz = g->dims[2];
  p.ox = g->origin[0];
  p.oy = g->origin[1];
  p.oz = g->origin[2];
  p.sx = g->spacing[0];
  p.sy = g->spacing[1];
  p.sz = g->spacing[2];
  p.E = d->n_elements;
  p.A = d->n_angles;
  p.T = d->n_samples;
  p.F = d->n_frames;
  p.fs = d->sampling_rate;
  p.c = bf->c;
  p.fc = bf->center_frequency;
  p.fnum = bf->f_number;
  p.interp = bf->interp_order;
  p.taps = bf->lowpass_taps;
  for (int a = 0; a < p.A; ++a) {
    double sina = std::sin(d->angles[a]), cosa = std::cos(d->angles[a]);
    double ref = std::numeric_limits<double>::infinity();
    for (int e = 0; e < p.E; ++e) ref = std::min(ref, pr->xyz[3 * e] * sina);
    p.ang[a] = AngleConst{sina, cosa, ref, d->t0[a]};
  }
  p.iq_row0 = 0;
  p.iq_rows = p.T + 2;
  plan_shape(P, iq_budget, p.T + 2);

  CK(cudaMalloc(&P.d_elem, sizeof(double) * 3 * p.E));
  CK(cudaMemcpy(P.d_elem, pr->xyz, sizeof(double) * 3 * p.E, cudaMemcpyHostToDevice));
  P.h_elem.assign(pr->xyz, pr->xyz + 3 * (size_t)p.E);
  p.elem = P.d_elem;
  std::vector<double2> car = carrier_table(d->t0, p.A, p.T, p.fc, p.fs);
  CK(cudaMalloc(&P.d_car, sizeof(double2) * car.size()));
  CK(cudaMemcpy(P.d_car, car.data(), sizeof(double2) * car.size(), cudaMemcpyHostToDevice));
  std::vector<double> h = lowpass(p.fc, p.fs, p.taps);
  std::vector<float> hf(h.begin(), h.end());
  P.hsum = 0.f;
  for (float v : hf) P.hsum += std::fabs(v);
  CK(cudaMalloc(&P.d_h, sizeof(float) * hf.size()));
  CK(cudaMemcpy(P.d_h, hf.data(), sizeof(float) * hf.size(), cudaMemcpyHostToDevice));

  unsigned long long* d_cnt;
  CK(cudaMalloc(&d_cnt, sizeof(unsigned long long)));
  CK(cudaMemset(d_cnt, 0, sizeof(unsigned long long)));
  size_t N = (size_t)p.nx * p.ny * p.nz;
  count_active_kernel<<<(unsigned)((N + 255) / 256), 256>>>(p, d_cnt);
  CK_LAUNCH();
  unsigned long long cnt = 0;
  CK(cudaMemcpy(&cnt, d_cnt, sizeof cnt, cudaMemcpyDeviceToHost));
  cudaFree(d_cnt);
  P.active_pairs = cnt * (uint64_t)p.A;
}

void free_plan(fqfg_das_plan_s* P) {
  if (!P) return;
  for (cudaEvent_t e : P->ev) cudaEventDestroy(e);
  P->ev.clear();
  cudaFree(P->d_elem);
  cudaFree(P->d_car);
  cudaFree(P->d_h);
}

// Accumulate the event times of the previous timed call (waits for it).
void harvest_timing(fqfg_das_plan_s& P) {
  if (P.ev_used == 0) return;
  for (int pass = 0; pass < P.ev_used; ++pass) {
    float t;
    CK(cudaEventSynchronize(P.ev[4 * pass + 3]));
    CK(cudaEventElapsedTime(&t, P.ev[4 * pass], P.ev[4 * pass + 1]));
    P.acc_demod_ms += t;
    CK(cudaEventElapsedTime(&t, P.ev[4 * pass + 2], P.ev[4 * pass + 3]));
    P.acc_das_ms += t;
  }
  P.acc_calls++;
  P.ev_used = 0;
}

// Padded IQ rows [row_lo, row_hi] (row = t + 1) that the DAS of z-planes
// [kb, ke) can read: the union over angles and elements of the conservative
// per-tile windows das2's producers use (same bounds, slab box instead of
// tile box, one extra row of margin).  With the f-number cut, a pair's range
// is at most (z - e_z) sqrt(1 + 1/(2F#)^2).
void slab_rows(const fqfg_das_plan_s& P, int kb, int ke, int& row_lo, int& row_hi) {
  const DasParams& p = P.p;
  const double x0 = p.ox, x1 = p.ox + (p.nx - 1) * p.sx;
  const double y0 = p.oy, y1 = p.oy + (p.ny - 1) * p.sy;
  const double z0 = p.oz + kb * p.sz, z1 = p.oz + (ke - 1) * p.sz;
  const std::vector<double>& el = P.h_elem;
  double lo = std::numeric_limits<double>::infinity(), hi = -lo;
  const double cone = p.fnum > 0.0 ? std::sqrt(1.0 + 1.0 / (4.0 * p.fnum * p.fnum)) : 0.0;
  for (int a = 0; a < p.A; ++a) {
    const AngleConst& ac = p.ang[a];
    const double tmin = (std::min(x0 * ac.sina, x1 * ac.sina) + z0 * ac.cosa - ac.ref) / p.c;
    const double tmax = (std::max(x0 * ac.sina, x1 * ac.sina) + z1 * ac.cosa - ac.ref) / p.c;
    for (int e = 0; e < p.E; ++e) {
      const double ex = el[3 * e], ey = el[3 * e + 1], ez = el[3 * e + 2];
      const double dxn = std::max({x0 - ex, ex - x1, 0.0}), dyn = std::max({y0 - ey, ey - y1, 0.0}),
                   dzn = std::max({z0 - ez, ez - z1, 0.0});
      const double dxf = std::max(std::fabs(x0 - ex), std::fabs(x1 - ex)),
                   dyf = std::max(std::fabs(y0 - ey), std::fabs(y1 - ey)),
                   dzf = std::max(std::fabs(z0 - ez), std::fabs(z1 - ez));
      double dmax = std::sqrt(dxf * dxf + dyf * dyf + dzf * dzf);
      if (p.fnum > 0.0) {
        if (z1 - ez < 0.0) continue;  // every voxel outside this element's aperture
        dmax = std::min(dmax, (z1 - ez) * cone);
      }
      const double dmin = std::sqrt(dxn * dxn + dyn * dyn + dzn * dzn);
      lo = std::min(lo, (tmin + dmin / p.c - ac.t0) * p.fs);
      hi = std::max(hi, (tmax + dmax / p.c - ac.t0) * p.fs);
    }
  }
  if (!(lo <= hi)) {
    row_lo = 1;
    row_hi = 0;  // nothing to demodulate
    return;
  }
  row_lo = (int)std::max(0.0, std::min((double)p.T + 1, std::floor(lo) - 3.0 + 1.0));
  row_hi = (int)std::max(0.0, std::min((double)p.T + 1, std::floor(hi) + 3.0 + 2.0));
}

// ---- the three launch steps of a frame pass (run_das and the
// reconstruction engine compose them) ----

// p: the plan's parameters with the pass buffer's row window (iq_row0,
// iq_rows) of the launch's slab.
//
// Demodulate pass frames [src.f_base, src.f_base + n) (frames >= nf of the
// pass are zeros) into IQ rows [row_lo, row_hi] of the pass buffer in
// d_work.  src.f_base is a multiple of 16 unless the launch starts the pass.
void demod_frames(fqfg_das_plan_s& P, const DasParams& p, const RfSrc& src, int n, int nf,
                  void* d_work, int row_lo, int row_hi, cudaStream_t st) {
  if (row_lo > row_hi || n <= 0) return;
  float2* stage = static_cast<float2*>(d_work);
  float2* iq = reinterpret_cast<float2*>(static_cast<char*>(d_work) + P.stage_bytes);
  if (P.tc) {
    // per-frame scale S_f from max |RF| of the frames, then mix + FIR into
    // the fp16 hi/lo layout of das_tc_kernel
    char* aux = reinterpret_cast<char*>(iq);
    unsigned* mx = reinterpret_cast<unsigned*>(aux);
    float* sc = reinterpret_cast<float*>(aux + 4 * (size_t)p.fpass);
    __half* iq16 = reinterpret_cast<__half*>(aux + P.tc_aux);
    const int fl = src.f_base;
    CK(cudaMemsetAsync(mx + fl, 0, sizeof(unsigned) * (size_t)n, st));
    {  // the bulk copy of the last element may read up to 4 chunks (x 2 planes) past the end
      // halves per plane: A E (TP / 4) chunks x fpass x 8
      const size_t plane = (size_t)2 * p.A * p.E * (size_t)((p.iq_rows + 3) & ~3) * p.fpass;
      CK(cudaMemsetAsync(iq16 + 2 * plane, 0, (size_t)8 * p.fpass * 16, st));
    }
    const int nv = std::min(n, nf - fl);
    if (nv > 0) {
      const size_t per = (size_t)src.rows * p.E;  // one (frame, angle) window
      const unsigned bx = (unsigned)std::max<size_t>(1, std::min<size_t>(8, per / 4096));
      rf_frame_absmax_kernel<<<dim3(bx, nv, p.A), 256, 0, st>>>(src, p.A, p.E, fl, mx);
      CK_LAUNCH();
    }
    tc_scale_kernel<<<(n + 127) / 128, 128, 0, st>>>(mx, P.hsum, fl, n, sc);
    CK_LAUNCH();
    const size_t fused_smem = fused_demod_smem(p.taps);
    smem_attr((void*)demod_fused_kernel<true, true>, fused_smem);
    smem_attr((void*)demod_fused_kernel<false, true>, fused_smem);
    const int TP = (p.iq_rows + 3) & ~3;
    dim3 g((n + kFusedG - 1) / kFusedG, (row_hi - row_lo + kFusedRB) / kFusedRB,
           p.A * ((p.E + 31) / 32));
    if (p.taps == 33)
      demod_fused_kernel<true, true><<<g, 256, fused_smem, st>>>(
          src, iq, P.d_car, P.d_h, p.T, p.E, p.A, p.taps, nf, p.fpass, row_lo, row_hi, p.iq_row0,
          p.iq_rows, iq16, sc, TP);
    else
      demod_fused_kernel<false, true><<<g, 256, fused_smem, st>>>(
          src, iq, P.d_car, P.d_h, p.T, p.E, p.A, p.taps, nf, p.fpass, row_lo, row_hi, p.iq_row0,
          p.iq_rows, iq16, sc, TP);
    CK_LAUNCH();
    return;
  }
  if (P.fused_demod) {
    const size_t fused_smem = fused_demod_smem(p.taps);
    smem_attr((void*)demod_fused_kernel<true>, fused_smem);
    smem_attr((void*)demod_fused_kernel<false>, fused_smem);
    dim3 g((n + kFusedG - 1) / kFusedG, (row_hi - row_lo + kFusedRB) / kFusedRB,
           p.A * ((p.E + 31) / 32));
    if (p.taps == 33)
      demod_fused_kernel<true><<<g, 256, fused_smem, st>>>(src, iq, P.d_car, P.d_h, p.T, p.E, p.A,
                                                           p.taps, nf, p.fpass, row_lo, row_hi,
                                                           p.iq_row0, p.iq_rows);
    else
      demod_fused_kernel<false><<<g, 256, fused_smem, st>>>(src, iq, P.d_car, P.d_h, p.T, p.E,
                                                            p.A, p.taps, nf, p.fpass, row_lo,
                                                            row_hi, p.iq_row0, p.iq_rows);
    CK_LAUNCH();
    return;
  }
  const int t_first = std::max(row_lo - 1, 0), t_last = std::min(row_hi - 1, p.T - 1);
  const int nv = std::min(n, nf - src.f_base);  // staged frames (the pack zero-fills the rest)
  if (t_first <= t_last && nv > 0) {
    const size_t fir_smem = (size_t)(kDemodTB + p.taps - 1) * 32 * sizeof(float2) +
                            p.taps * sizeof(float);
    smem_attr((void*)demod_fir_kernel, fir_smem);
    const int b0 = t_first / kDemodTB, b1 = t_last / kDemodTB;
    dim3 g1(b1 - b0 + 1, (p.E + 31) / 32, nv * p.A);
    demod_fir_kernel<<<g1, 256, fir_smem, st>>>(src, stage, P.d_car, P.d_h, p.T, p.E, p.A,
                                                p.taps, b0);
    CK_LAUNCH();
  }
}

// Two-kernel form: transpose the staged pass into the DAS layout (after every
// demod_frames of the pass); nothing to do for the fused demodulation.
void demod_finish(fqfg_das_plan_s& P, const DasParams& p, int nf, void* d_work, int row_lo,
                  int row_hi, cudaStream_t st) {
  if (P.tc || P.fused_demod || row_lo > row_hi) return;
  float2* stage = static_cast<float2*>(d_work);
  float2* iq = reinterpret_cast<float2*>(static_cast<char*>(d_work) + P.stage_bytes);
  const size_t pack_smem = (size_t)p.fpass * 33 * sizeof(float2);
  smem_attr((void*)demod_pack_kernel, pack_smem);
  dim3 g2(row_hi - row_lo + 1, (p.E + 31) / 32, p.A);
  demod_pack_kernel<<<g2, 256, pack_smem, st>>>(stage, iq, p.T, p.E, p.A, nf, p.fpass, row_lo,
                                                p.iq_row0, p.iq_rows);
  CK_LAUNCH();
}

PFN_cuTensorMapEncodeTiled tensor_map_encoder();

// Tensor-core DAS launch (das_tc.cu) over the fp16 IQ in row chunks.
void das_tc_pass(fqfg_das_plan_s& P, const DasParams& p, int pass, int kb, int ke,
                 const float2* iq, float2* d_x, size_t x_v0, size_t x_n,
                 unsigned long long* d_counters, cudaStream_t st) {
  const char* aux = reinterpret_cast<const char*>(iq);
  const float* sc = reinterpret_cast<const float*>(aux + 4 * (size_t)p.fpass);
  const void* iq16 = aux + P.tc_aux;
  smem_attr((void*)das_tc_kernel, P.smem);
  DasLaunch L{};
  L.TX = P.TX;
  L.TY = P.TY;
  L.TZ = P.TZ;
  L.tiles_x = (p.nx + P.TX - 1) / P.TX;
  L.tiles_y = (p.ny + P.TY - 1) / P.TY;
  const int tiles_z = (ke - kb + P.TZ - 1) / P.TZ;
  L.kbeg = kb;
  L.kend = ke;
  L.pass = pass;
  L.rcap = P.rcap;  // X slots
  L.kblocks = P.d_kblocks;
  L.x_v0 = (long long)x_v0;
  L.x_n = (long long)x_n;
  const size_t n_tiles = (size_t)L.tiles_x * L.tiles_y * tiles_z;
  require(n_tiles < (1u << 31), "grid too large");
  das_tc_kernel<<<(unsigned)n_tiles, kTcWarps * 32, P.smem, st>>>(
      p, L, static_cast<const __half*>(iq16), sc, d_x, d_counters);
  CK_LAUNCH();
  g_launches.fetch_add(1);
}

// The DAS of pass `pass` for z-planes [kb, ke) from the IQ pass buffer into
// d_x, which holds grid voxels [x_v0, x_v0 + x_n) as [F][x_n].
void das_pass(fqfg_das_plan_s& P, const DasParams& p, int pass, int kb, int ke, void* d_work,
              float2* d_x, size_t x_v0, size_t x_n, unsigned long long* d_counters,
              cudaStream_t st) {
  if (kb >= ke) return;
  const float2* iq =
      reinterpret_cast<const float2*>(static_cast<const char*>(d_work) + P.stage_bytes);
  if (P.tc) {
    das_tc_pass(P, p, pass, kb, ke, iq, d_x, x_v0, x_n, d_counters, st);
    return;
  }
  void* kfn = pick_das2(P.J, P.VPW, P.NW, P.EB, P.NS, P.PW);
  smem_attr(kfn, P.smem);
  DasLaunch L;
  L.TX = P.TX;
  L.TY = P.TY;
  L.TZ = P.TZ;
  L.tiles_x = (p.nx + P.TX - 1) / P.TX;
  L.tiles_y = (p.ny + P.TY - 1) / P.TY;
  const int tiles_z = (ke - kb + P.TZ - 1) / P.TZ;
  L.kbeg = kb;
  L.kend = ke;
  L.rcap = P.rcap;
  L.pass = pass;
  L.x_v0 = (long long)x_v0;
  L.x_n = (long long)x_n;
  const size_t n_tiles = (size_t)L.tiles_x * L.tiles_y * tiles_z;
  require(n_tiles < (1u << 31), "grid too large");
  void* args[] = {(void*)&p, (void*)&L, (void*)&iq, (void*)&d_x, (void*)&d_counters};
  CK(cudaLaunchKernel(kfn, dim3((unsigned)n_tiles), dim3(32 * (P.NW + P.PW)), args, P.smem, st));
  g_launches.fetch_add(1);
}

// Demod + DAS of every pass for z-planes [kb, ke) into d_x, which holds grid
// voxels [x_v0, x_v0 + x_n) as [F][x_n] (x_n = 0: the whole grid).
void run_das(fqfg_das_plan_s& P, const float* d_rf, int kb, int ke, float2* d_x,
             void* d_work, unsigned long long* d_counters, cudaStream_t st, size_t x_v0 = 0,
             size_t x_n = 0) {
  const DasParams& p = P.p;
  require(kb >= 0 && ke <= p.nz && kb <= ke, "z-slab [%d, %d) outside the grid", kb, ke);
  if (kb == ke) return;
  const size_t N = (size_t)p.nx * p.ny * p.nz;
  if (x_n == 0) x_v0 = 0, x_n = N;
  require(x_v0 + x_n <= N && (size_t)kb * p.nx * p.ny >= x_v0 &&
              (size_t)ke * p.nx * p.ny <= x_v0 + x_n,
          "output range [%zu, %zu) does not hold z-slab [%d, %d)", x_v0, x_v0 + x_n, kb, ke);
  int row_lo = 0, row_hi = p.T + 1;
  // Only the IQ rows some voxel of the slab can read are demodulated (the
  // whole grid included: the samples before the earliest echo and after the
  // latest never reach the output).
  slab_rows(P, kb, ke, row_lo, row_hi);
  DasParams pp = p;  // the pass buffer holds the slab's readable rows only
  if (row_lo <= row_hi) pp.iq_row0 = row_lo, pp.iq_rows = row_hi - row_lo + 1;
  if (P.timing) {
    harvest_timing(P);
    while (P.ev.size() < (size_t)4 * p.npass) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      P.ev.push_back(e);
    }
    P.ev_used = p.npass;
  }
  for (int pass = 0; pass < p.npass; ++pass) {
    const int f0 = pass * p.fpass;
    const int nf = std::min(p.fpass, p.F - f0);
    RfSrc src{d_rf + (size_t)f0 * p.A * p.T * p.E, (long long)p.A * p.T * p.E,
              (long long)p.T * p.E, 0, p.T, 0};
    if (P.timing) CK(cudaEventRecord(P.ev[4 * pass], st));
    demod_frames(P, pp, src, p.fpass, nf, d_work, row_lo, row_hi, st);
    demod_finish(P, pp, nf, d_work, row_lo, row_hi, st);
    if (P.timing) CK(cudaEventRecord(P.ev[4 * pass + 1], st));
    if (P.timing) CK(cudaEventRecord(P.ev[4 * pass + 2], st));
    das_pass(P, pp, pass, kb, ke, d_work, d_x, x_v0, x_n, d_counters, st);
    if (P.timing) CK(cudaEventRecord(P.ev[4 * pass + 3], st));
  }
}

// FP64 Gram tile: the TB whose padded upper triangle nb (nb + 1) / 2 TB^2 is
// smallest (ties -> larger TB).
int gram_tile(int F) {
  int best = 64;
  double cost = 1e300;
  for (int tb : {64, 48, 40, 32}) {
    const double nb = (F + tb - 1) / tb;
    const double c = nb * (nb + 1) / 2 * tb * tb;
    if (c < cost) cost = c, best = tb;
  }
  return best;
}

size_t gram_splits(int F) {
  const int TB = gram_tile(F);
  const int nb = (F + TB - 1) / TB;
  const int blocks = nb * (nb + 1) / 2;
  // two waves of resident CTAs (gram_min_ctas per SM); the split-K partials
  // cost splits x F^2 x 16 B of scratch and one reduction read
  const int per_sm = gram_min_ctas(TB);
  return (size_t)std::max(1, std::min(256, 2 * 148 * per_sm / blocks));
}

template <int TB>
void launch_gram_partial(const float2* d_x, int F, size_t N, size_t v0, size_t v1,
                         double2* work, int blocks, int splits, cudaStream_t st) {
  smem_attr((void*)gram_partial_kernel<TB>, gram_smem(TB));
  gram_partial_kernel<TB><<<dim3(blocks, (unsigned)splits), gram_threads(TB), gram_smem(TB), st>>>(
      d_x, F, N, v0, v1, work);
}

void run_gram_fp64(const float2* d_x, int F, size_t N, size_t v0, size_t v1, double2* d_g,
                   void* d_work, int accumulate, cudaStream_t st) {
  const int TB = gram_tile(F);
  const int nb = (F + TB - 1) / TB;
  const int blocks = nb * (nb + 1) / 2;
  const int splits = (int)gram_splits(F);
  double2* work = static_cast<double2*>(d_work);
  switch (TB) {
    case 64: launch_gram_partial<64>(d_x, F, N, v0, v1, work, blocks, splits, st); break;
    case 48: launch_gram_partial<48>(d_x, F, N, v0, v1, work, blocks, splits, st); break;
    case 40: launch_gram_partial<40>(d_x, F, N, v0, v1, work, blocks, splits, st); break;
    default: launch_gram_partial<32>(d_x, F, N, v0, v1, work, blocks, splits, st); break;
  }
  CK_LAUNCH();
  size_t n = (size_t)F * F;
  gram_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(work, F, splits, d_g,
                                                                   accumulate, TB);
  CK_LAUNCH();
}

void run_gram(const float2* d_x, int F, size_t N, size_t v0, size_t v1, double2* d_g,
              void* d_work, int accumulate, cudaStream_t st) {
  run_gram_fp64(d_x, F, N, v0, v1, d_g, d_work, accumulate, st);
}

// ---- the tensor-core Gram (gram_i8.cu) ----

PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    require(p != nullptr && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

// Tiles of 128 frames (A rows) x <= 64 frames (B rows) covering the F x F
// square (the antisymmetric Im G needs P and P^T): M tiles start at
// min(128 t, Fp - 128), so none runs past the padded frame count.
I8Gram i8_tiles(int F) {
  require(F >= 1 && F <= 1024, "tensor-core Gram supports 1..1024 frames");
  I8Gram g{};
  g.F = F;
  const int Fp = (F + 15) / 16 * 16;
  const int mt = (F + kI8TileM - 1) / kI8TileM, nt = (F + kI8TileN - 1) / kI8TileN;
  g.ntile = mt * nt;
  require(g.ntile <= kI8MaxTiles, "tensor-core Gram: %d tiles exceed %d", g.ntile, kI8MaxTiles);
  for (int a = 0; a < mt; ++a)
    for (int b = 0; b < nt; ++b) {
      const int t = a * nt + b;
      g.m0[t] = Fp <= kI8TileM ? 0 : std::min(kI8TileM * a, Fp - kI8TileM);
      g.n0[t] = kI8TileN * b;
      g.nn[t] = std::min(kI8TileN, Fp - g.n0[t]);
    }
  return g;
}

// Digit batches: Q holds 4 F bytes per voxel; whole ensembles up to 2^21
// voxels at F <= 256 (config C in one batch), smaller batches above.
size_t i8_batch(int F) { return F <= 256 ? (size_t)1 << 21 : (size_t)1 << 20; }
size_t i8_q_bytes(int F, size_t batch) { return (size_t)4 * F * 128 * ((batch + 63) / 64); }
size_t i8_part_bytes(int F, size_t batch) {
  const I8Gram g = i8_tiles(F);
  const size_t nsplit = (batch + kI8SplitVox - 1) / kI8SplitVox;
  return nsplit * g.ntile * (size_t)kI8TileM * kI8TileN * sizeof(double2);
}
size_t i8_amax_bytes(int F) { return ((size_t)4 * F + 255) / 256 * 256; }
size_t gram_tc_work_bytes(int F) {
  return i8_amax_bytes(F) + (i8_q_bytes(F, i8_batch(F)) + 255) / 256 * 256 +
         i8_part_bytes(F, i8_batch(F));
}

CUtensorMap i8_map(const void* q, int F, size_t kb, int rows) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)kb, (cuuint64_t)F, 4};
  const cuuint64_t strides[2] = {(cuuint64_t)kb, (cuuint64_t)F * kb};
  const cuuint32_t box[3] = {128, (cuuint32_t)rows, 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(q), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (Gram digits) failed: %d", (int)r);
  return m;
}

// G (+)= X^H X over voxels [v0, v1) of x [F][N] on the tensor cores (int8
// digit planes of voxel batches; see gram_i8.cu).  d_work: gram_tc_work_bytes(F).
void run_gram_tc(const float2* d_x, int F, size_t N, size_t v0, size_t v1, double2* d_g,
                 void* d_work, int accumulate, cudaStream_t st) {
  I8Gram g = i8_tiles(F);
  char* w = static_cast<char*>(d_work);
  unsigned* amax = reinterpret_cast<unsigned*>(w);
  unsigned char* Q = reinterpret_cast<unsigned char*>(w + i8_amax_bytes(F));
  const size_t batch = i8_batch(F);
  double2* part = reinterpret_cast<double2*>(w + i8_amax_bytes(F) +
                                             (i8_q_bytes(F, batch) + 255) / 256 * 256);
  g.amax = amax;
  const size_t len = v1 > v0 ? v1 - v0 : 0;
  if (len == 0) {
    if (!accumulate) CK(cudaMemsetAsync(d_g, 0, (size_t)F * F * sizeof(double2), st));
    return;
  }
  CK(cudaMemsetAsync(amax, 0, sizeof(unsigned) * F, st));
  {
    const unsigned gx =
        (unsigned)std::max<size_t>(1, std::min<size_t>(4 * 148 * 8 / F + 1, (len + 8191) / 8192));
    gram_amax_kernel<<<dim3(gx, F), 256, 0, st>>>(d_x, N, v0, v1, amax);
    CK_LAUNCH();
  }
  smem_attr((void*)gram_i8_mma_kernel, kI8Smem);
  bool first = true;
  for (size_t b0 = 0; b0 < len; b0 += batch) {
    const size_t nb = std::min<size_t>(batch, len - b0);
    const size_t kb = 128 * ((nb + 63) / 64);
    const size_t octs = (nb + 63) / 64 * 8;
    gram_i8_split_kernel<<<dim3((unsigned)((octs + 255) / 256), F), 256, 0, st>>>(
        d_x, N, v0 + b0, nb, amax, F, kb, reinterpret_cast<unsigned*>(Q));
    CK_LAUNCH();
    g.nvox = nb;
    g.nsplit = (int)((nb + kI8SplitVox - 1) / kI8SplitVox);
    const CUtensorMap ma = i8_map(Q, F, kb, kI8TileM), mb = i8_map(Q, F, kb, kI8TileN);
    gram_i8_mma_kernel<<<(unsigned)(g.ntile * g.nsplit), kI8Threads, kI8Smem, st>>>(ma, mb, g,
                                                                                   part);
    CK_LAUNCH();
    const size_t n = (size_t)F * F;
    gram_i8_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, g, d_g,
                                                                      (accumulate || !first) ? 1 : 0);
    CK_LAUNCH();
    first = false;
  }
}

size_t eig_work_bytes(int F) {
  size_t f = (size_t)F;
  size_t max_rot = 64 * f * f + 64, max_seq = 64 * f + 64;
  return f * f * sizeof(double) /*Z*/ + f * f * sizeof(double2) /*V unsorted*/ +
         4 * f * sizeof(double) + f * sizeof(double2) + max_rot * sizeof(double2) +
         max_seq * sizeof(int3) + 1024;
}

constexpr int kEigMaxF = 1024;

// Householder tridiagonalisation + QL (eig2.cu).  d_g is destroyed.
void run_eig(double2* d_g, int F, double* d_w, double2* d_v, void* d_work, cudaStream_t st) {
  require(F >= 1 && F <= kEigMaxF, "eigensolve supports 1..%d frames", kEigMaxF);
  size_t f = (size_t)F;
  size_t max_rot = 64 * f * f + 64, max_seq = 64 * f + 64;
  char* p = static_cast<char*>(d_work);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  double* Z = reinterpret_cast<double*>(take(f * f * sizeof(double)));
  double2* Vu = reinterpret_cast<double2*>(take(f * f * sizeof(double2)));
  double* d = reinterpret_cast<double*>(take(f * sizeof(double)));
  double* e = reinterpret_cast<double*>(take(f * sizeof(double)));
  double2* tau = reinterpret_cast<double2*>(take(f * sizeof(double2)));
  int* status = reinterpret_cast<int*>(take(16));
  int3* seq = reinterpret_cast<int3*>(take(max_seq * sizeof(int3)));
  double2* rot = reinterpret_cast<double2*>(take(max_rot * sizeof(double2)));

  size_t tri_smem = 2 * f * sizeof(double2) + 80 * sizeof(double);
  smem_attr((void*)tridiag_kernel, tri_smem);
  tridiag_kernel<<<1, kTriThreads, tri_smem, st>>>(d_g, F, d, e, tau);
  CK_LAUNCH();
  tql2_kernel<<<1, 32, 2 * f * sizeof(double), st>>>(d, e, F, rot, seq, (int)max_rot,
                                                     (int)max_seq, status);
  CK_LAUNCH();
  unsigned nb = (unsigned)((F + 31) / 32);
  size_t zr_smem = 32 * (f + 1) * sizeof(double);
  smem_attr((void*)zrot_kernel, zr_smem);
  zrot_kernel<<<nb, 32, zr_smem, st>>>(F, rot, seq, status, Z);
  CK_LAUNCH();
  size_t bt_smem = f * 33 * sizeof(double2);
  smem_attr((void*)backtrans_kernel, bt_smem);
  backtrans_kernel<<<nb, 32, bt_smem, st>>>(d_g, F, tau, Z, Vu);
  CK_LAUNCH();
  eig_sort_kernel<<<nb, 32, 0, st>>>(d, Vu, F, d_w, d_v);
  CK_LAUNCH();
}

// Modes whose eigenvectors the rank-form projection reads (run_project):
// the band [lo, hi] or its complement, whichever is smaller.
std::vector<int> projection_modes(int F, int lo, int hi) {
  const int rb = hi - lo + 1, rc = F - rb;
  const bool complement = rc < rb;
  std::vector<int> modes;
  for (int j = 0; j < F; ++j) {
    const bool in_band = j >= lo - 1 && j < hi;
    if (in_band != complement) modes.push_back(j);
  }
  return modes;
}

// Eigenvalues (descending) and the eigenvectors the projection of band
// [lo, hi] reads.  With <= 8 such vectors: tridiagonalisation, bisection
// and inverse iteration (eig2.cu) instead of the full QL + back-transform
// (14 ms -> ~3 ms at F = 200); other columns of d_v are left unset.
void run_eig_band(double2* d_g, int F, int lo, int hi, double* d_w, double2* d_v, void* d_work,
                  cudaStream_t st) {
  const std::vector<int> modes = projection_modes(F, lo, hi);
  const int r = (int)modes.size();
  if (r > kInvitMax || F > kInvitMaxF) {
    run_eig(d_g, F, d_w, d_v, d_work, st);
    return;
  }
  size_t f = (size_t)F;
  char* p = static_cast<char*>(d_work);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) / 256 * 256;
    return q;
  };
  double* d = reinterpret_cast<double*>(take(f * sizeof(double)));
  double* e = reinterpret_cast<double*>(take(f * sizeof(double)));
  double2* tau = reinterpret_cast<double2*>(take(f * sizeof(double2)));
  int* d_modes = reinterpret_cast<int*>(take(kInvitMax * sizeof(int)));
  double* z = reinterpret_cast<double*>(take(f * kInvitMax * sizeof(double)));
  double* scr = reinterpret_cast<double*>(take(6 * f * kInvitMax * sizeof(double)));
  size_t tri_smem = 2 * f * sizeof(double2) + 80 * sizeof(double);
  smem_attr((void*)tridiag_kernel, tri_smem);
  tridiag_kernel<<<1, kTriThreads, tri_smem, st>>>(d_g, F, d, e, tau);
  CK_LAUNCH();
  bisect_kernel<<<(F + 127) / 128, 128, 2 * f * sizeof(double), st>>>(d, e, F, d_w);
  CK_LAUNCH();
  if (r == 0) return;
  static thread_local std::vector<int> pinned_modes;  // stays alive for the async copy
  pinned_modes = modes;
  CK(cudaMemcpyAsync(d_modes, pinned_modes.data(), r * sizeof(int), cudaMemcpyHostToDevice, st));
  invit_kernel<<<1, 32, 0, st>>>(d, e, F, d_w, d_modes, r, z, scr);
  CK_LAUNCH();
  const size_t bt_smem = f * r * sizeof(double2);
  smem_attr((void*)backtrans_sel_kernel, bt_smem);
  backtrans_sel_kernel<<<1, 32 * r, bt_smem, st>>>(d_g, F, tau, z, r, d_modes, d_v);
  CK_LAUNCH();
}

// Band projection + PD.  d_scratch: >= F*F*16 + F*8*16 + 64 bytes.
void run_project(const float2* d_x, int F, size_t N, size_t v0, size_t v1, const double2* d_v,
                 int lo, int hi, float2* d_y, double* d_pd, void* d_scratch, cudaStream_t st) {
  int rb = hi - lo + 1, rc = F - rb;
  bool complement = rc < rb;
  int r = complement ? rc : rb;
  size_t len = v1 - v0;
  if (len == 0) return;
  if (r == 0) {  // full band: identity (complement of nothing)
    if (d_y)
      for (int f = 0; f < F; ++f)
        CK(cudaMemcpyAsync(d_y + (size_t)f * N + v0, d_x + (size_t)f * N + v0,
                           len * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    if (d_pd) {
      // PD of X restricted to the range.
      power_doppler_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(d_x, F, N, v0, v1,
                                                                          d_pd);
      CK_LAUNCH();
    }
    return;
  }
  if (r <= kProjMaxR) {
    std::vector<int> modes;
    for (int j = 0; j < F; ++j) {
      bool in_band = j >= lo - 1 && j < hi;
      if (in_band != complement) modes.push_back(j);
    }
    int* d_modes = static_cast<int*>(d_scratch);
    double2* vm = reinterpret_cast<double2*>(static_cast<char*>(d_scratch) + 64);
    CK(cudaMemcpyAsync(d_modes, modes.data(), sizeof(int) * modes.size(), cudaMemcpyHostToDevice,
                       st));
    int R = r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : 8;
    select_modes_kernel<<<1, 256, 0, st>>>(d_v, F, d_modes, r, R, vm);
    CK_LAUNCH();
    size_t smem = (size_t)F * R * sizeof(double2);
    unsigned grid = (unsigned)((len + 255) / 256);
#define LAUNCH_R(RR)                                                                        \
  case RR:                                                                                 \
    smem_attr((void*)project_rank_kernel<RR>, smem);                                       \
    project_rank_kernel<RR><<<grid, 256, smem, st>>>(d_x, F, N, v0, v1, vm, complement, d_y, \
                                                     d_pd);                                \
    break;
    switch (R) {
      LAUNCH_R(1)
      LAUNCH_R(2)
      LAUNCH_R(4)
      LAUNCH_R(8)
    }
#undef LAUNCH_R
    CK_LAUNCH();
    return;
  }
  double2* P = reinterpret_cast<double2*>(static_cast<char*>(d_scratch) + 64);
  size_t n = (size_t)F * F;
  projector_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_v, F, lo, hi, P);
  CK_LAUNCH();
  size_t smem = (size_t)F * kProjFC * sizeof(double2);
  smem_attr((void*)project_full_kernel, smem);
  project_full_kernel<<<(unsigned)((len + 127) / 128), 128, smem, st>>>(d_x, F, N, v0, v1, P, d_y,
                                                                      d_pd);
  CK_LAUNCH();
}

void check_filter(int F, size_t N, int lo, int hi) {
  require(F >= 1, "svd_filter needs a nonempty ensemble");
  require(N > 0, "svd_filter needs a nonempty grid");
  require(F >= 2, "svd_filter needs at least two frames");
  require((size_t)F <= N, "svd_filter needs at least as many voxels as frames");
  require(lo >= 1 && lo <= hi && hi <= F,
          "retained band must satisfy 1 <= lo <= hi <= frames, got [%d, %d] with %d frames", lo,
          hi, F);
  require(F <= kEigMaxF, "svd_filter supports at most %d frames", kEigMaxF);
}

size_t filter_scratch_bytes(int F) {
  return (size_t)F * F * sizeof(double2) + (size_t)F * 8 * sizeof(double2) + 128;
}

// SvdReport::mode_correlation (svd.cpp:55-75) from V and sigma on device.
void run_mode_correlation(const float2* d_x, int F, size_t N, const double2* d_v,
                          const std::vector<double>& sigma, double* h_corr, cudaStream_t st) {
  size_t nb = std::min<size_t>((N + 4095) / 4096, 64);
  size_t chunk = (N + nb - 1) / nb;
  nb = (N + chunk - 1) / chunk;
  size_t m_bytes = (size_t)F * N * sizeof(double);
  size_t part_bytes = nb * (size_t)F * F * sizeof(double);
  char* buf = static_cast<char*>(tl_corr.get(m_bytes + part_bytes + 2 * F * sizeof(double) + 512));
  double* d_m = reinterpret_cast<double*>(buf);
  double* d_part = reinterpret_cast<double*>(buf + m_bytes);
  double* d_inv = reinterpret_cast<double*>(buf + m_bytes + part_bytes);
  double* d_mean = d_inv + F;
  std::vector<double> inv(F);
  for (int j = 0; j < F; ++j) inv[j] = sigma[j] > 0.0 ? 1.0 / sigma[j] : 0.0;
  CK(cudaMemcpyAsync(d_inv, inv.data(), F * sizeof(double), cudaMemcpyHostToDevice, st));
  size_t smem = (size_t)F * kMagModes * sizeof(double2);
  smem_attr((void*)mode_mag_kernel, smem);
  mode_mag_kernel<<<dim3((unsigned)((N + 255) / 256), (F + kMagModes - 1) / kMagModes), 256, smem,
                    st>>>(d_x, F, N, d_v, d_inv, d_m);
  CK_LAUNCH();
  col_sum_kernel<<<dim3((unsigned)nb, F), 256, 0, st>>>(d_m, F, N, chunk, d_part);
  CK_LAUNCH();
  std::vector<double> part(nb * (size_t)F);
  CK(cudaMemcpyAsync(part.data(), d_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<double> mean(F, 0.0);
  for (size_t b = 0; b < nb; ++b)
    for (int j = 0; j < F; ++j) mean[j] += part[b * F + j];
  for (int j = 0; j < F; ++j) mean[j] /= (double)N;
  CK(cudaMemcpyAsync(d_mean, mean.data(), F * sizeof(double), cudaMemcpyHostToDevice, st));
  int tb = (F + 31) / 32;
  centred_cov_kernel<<<dim3((unsigned)nb, tb, tb), 256, 0, st>>>(d_m, F, N, chunk, d_mean, d_part);
  CK_LAUNCH();
  std::vector<double> cp(nb * (size_t)F * F);
  CK(cudaMemcpyAsync(cp.data(), d_part, cp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<double> cov((size_t)F * F, 0.0);
  for (size_t b = 0; b < nb; ++b)
    for (size_t i = 0; i < (size_t)F * F; ++i) cov[i] += cp[b * F * F + i];
  std::vector<double> sd(F);
  for (int j = 0; j < F; ++j) sd[j] = std::sqrt(cov[(size_t)j * F + j] / (double)N);
  for (int i = 0; i < F; ++i) {
    h_corr[(size_t)i * F + i] = 1.0;
    for (int j = i + 1; j < F; ++j) {
      double den = sd[i] * sd[j], r = 0.0;
      if (den > 0.0) r = cov[(size_t)i * F + j] / ((double)N * den);
      h_corr[(size_t)i * F + j] = r;
      h_corr[(size_t)j * F + i] = r;
    }
  }
}

// Gram + eigensolve + projection/PD of a resident ensemble.
void run_filter(const float2* d_x, int F, size_t N, int lo, int hi, float2* d_y, double* d_pd,
                double* h_sigma, cudaStream_t st, double* h_corr = nullptr) {
  size_t gsz = (size_t)F * F * sizeof(double2);
  char* small = static_cast<char*>(
      tl_gram.get(2 * gsz + F * sizeof(double) + filter_scratch_bytes(F) + 1024));
  double2* d_g = reinterpret_cast<double2*>(small);
  double2* d_v = reinterpret_cast<double2*>(small + gsz);
  double* d_w = reinterpret_cast<double*>(small + 2 * gsz);
  void* scratch = small + 2 * gsz + ((F * sizeof(double) + 255) / 256) * 256;
  void* d_vw = tl_eig.get(std::max(eig_work_bytes(F), gsz));
  void* work = tl_work.get(gram_splits(F) * gsz);
  run_gram(d_x, F, N, 0, N, d_g, work, 0, st);
  // Nonzero check (svd.cpp:42): trace of the Gram = ||X||_F^2.
  std::vector<double2> g((size_t)F * F);
  CK(cudaMemcpyAsync(g.data(), d_g, gsz, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double tr = 0.0;
  for (int i = 0; i < F; ++i) tr += g[(size_t)i * F + i].x;
  require(tr > 0.0, "svd_filter needs a nonzero ensemble");
  if (h_corr)
    run_eig(d_g, F, d_w, d_v, d_vw, st);  // the report needs every mode's vector
  else
    run_eig_band(d_g, F, lo, hi, d_w, d_v, d_vw, st);
  if (h_sigma || h_corr) {
    std::vector<double> w(F), sg(F);
    CK(cudaMemcpyAsync(w.data(), d_w, F * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int j = 0; j < F; ++j) sg[j] = std::sqrt(std::max(w[j], 0.0));
    if (h_sigma) std::copy(sg.begin(), sg.end(), h_sigma);
    if (h_corr) run_mode_correlation(d_x, F, N, d_v, sg, h_corr, st);
  }
  if (d_y || d_pd) run_project(d_x, F, N, 0, N, d_v, lo, hi, d_y, d_pd, scratch, st);
}

// ------------------------------------------------ display and scoring --

thread_local DevBuf tl_disp_a, tl_disp_b, tl_disp_c, tl_disp_w, tl_disp_pk;

unsigned disp_blocks(size_t n) {
  return (unsigned)std::max<size_t>(1, (n + kDispThreads - 1) / kDispThreads);
}

// out = render_db(in) on device (render.cpp:44-68).
void run_render_db(const double* d_in, size_t n, double dr_db, bool power, double* d_out,
                   cudaStream_t st) {
  auto* peak = static_cast<unsigned long long*>(tl_disp_pk.get(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(peak, 0, sizeof(unsigned long long), st));
  peak_abs_kernel<<<std::min(disp_blocks(n), 1184u), kDispThreads, 0, st>>>(d_in, n, peak);
  CK_LAUNCH();
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, peak, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double pk;
  std::memcpy(&pk, &h, sizeof(pk));
  require(pk > 0.0, "render_db needs a nonzero volume");
  render_db_kernel<<<disp_blocks(n), kDispThreads, 0, st>>>(d_in, n, peak, power ? 10.0 : 20.0,
                                                             dr_db, d_out);
  CK_LAUNCH();
}

// MSE / PSNR / mean SSIM of two device images (metrics.cpp:24-101).
void run_metrics(const double* d_a, const double* d_b, const int* dims, double* out3,
                 cudaStream_t st) {
  const size_t n = (size_t)dims[0] * dims[1] * dims[2];
  const unsigned nb = std::min(disp_blocks(n), 1024u);
  double* part = static_cast<double*>(tl_disp_c.get(2048 * sizeof(double)));
  sqdiff_kernel<<<nb, kDispThreads, 0, st>>>(d_a, d_b, n, part);
  CK_LAUNCH();
  sum_kernel<<<1, kDispThreads, 0, st>>>(part, nb, part + 1024);
  CK_LAUNCH();
  // Window per axis: the largest odd size <= min(11, dim), Gaussian taps
  // (sigma 1.5) normalised jointly -- built exactly as metrics.cpp:24-49.
  int win[3], half[3];
  std::vector<double> taps[3];
  for (int ax = 0; ax < 3; ++ax) {
    int w = std::min(11, dims[ax]);
    if (w % 2 == 0) --w;
    win[ax] = w;
    half[ax] = w / 2;
    taps[ax].resize(w);
    for (int t = 0; t < w; ++t) {
      double d = t - half[ax];
      taps[ax][t] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    }
  }
  std::vector<double> weight((size_t)win[0] * win[1] * win[2]);
  double wsum = 0.0;
  for (int dk = 0; dk < win[2]; ++dk)
    for (int dj = 0; dj < win[1]; ++dj)
      for (int di = 0; di < win[0]; ++di) {
        double w = taps[0][di] * taps[1][dj] * taps[2][dk];
        weight[di + (size_t)win[0] * (dj + (size_t)win[1] * dk)] = w;
        wsum += w;
      }
  for (double& w : weight) w /= wsum;
  SsimGeom g;
  g.nx = dims[0], g.ny = dims[1], g.nz = dims[2];
  g.hx = half[0], g.hy = half[1], g.hz = half[2];
  g.wx = win[0], g.wy = win[1], g.wz = win[2];
  g.vx = dims[0] - 2 * half[0], g.vy = dims[1] - 2 * half[1], g.vz = dims[2] - 2 * half[2];
  const size_t nvalid = (size_t)g.vx * g.vy * g.vz;
  double* d_w = static_cast<double*>(tl_disp_w.get(weight.size() * sizeof(double)));
  CK(cudaMemcpyAsync(d_w, weight.data(), weight.size() * sizeof(double), cudaMemcpyHostToDevice,
                     st));
  double* local = static_cast<double*>(tl_disp_b.get(nvalid * sizeof(double)));
  ssim_kernel<<<disp_blocks(nvalid), kDispThreads, weight.size() * sizeof(double), st>>>(
      d_a, d_b, d_w, g, local);
  CK_LAUNCH();
  const unsigned nb2 = std::min(disp_blocks(nvalid), 1024u);
  sum_kernel<<<nb2, kDispThreads, 0, st>>>(local, nvalid, part);
  CK_LAUNCH();
  sum_kernel<<<1, kDispThreads, 0, st>>>(part, nb2, part + 1025);
  CK_LAUNCH();
  double h[2];
  CK(cudaMemcpyAsync(h, part + 1024, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out3[0] = h[0] / (double)n;
  out3[1] = out3[0] > 0.0 ? 10.0 * std::log10(1.0 / out3[0])
                          : std::numeric_limits<double>::infinity();
  out3[2] = h[1] / (double)nvalid;
}

size_t dims_points(const int* dims) {
  require(dims != nullptr, "image dims missing");
  for (int a = 0; a < 3; ++a) require(dims[a] > 0, "image dims must be positive");
  return (size_t)dims[0] * dims[1] * dims[2];
}

// ------------------------------------------------------- RF synthesis --

struct RfsBand {
  int T = 0, j_lo = 0, j_hi = 0;
  double df = 0.0, sigma = 0.0;
  int bins() const { return j_hi - j_lo + 1; }
};

void rf_validate_transducer(const fqfg_transducer* t) {  // transducer.cpp:10-24
  require(t && t->n_elements > 0 && t->xyz, "transducer has no elements");
  require(t->half_width > 0.0, "element half-width must be positive");
  require(t->subelements >= 1, "sub-element count must be at least 1");
  require(t->pitch > 0.0, "pitch must be positive");
  require(t->center_frequency > 0.0, "center frequency must be positive");
  require(t->fractional_bandwidth > 0.0 && t->fractional_bandwidth < 2.0,
          "fractional bandwidth must lie in (0, 2)");
  if (t->elevation_height > 0.0) {
    require(t->elevation_focus > 0.0, "elevation focus must be positive when a lens is present");
    require(t->elevation_aperture_factor > 0.0, "elevation aperture factor must be positive");
    require(t->elevation_core_weight >= 0.0 && t->elevation_tail_weight >= 0.0,
            "elevation weights must be nonnegative");
  }
}

RfsBand rf_passband(const fqfg_transducer* t, const fqfg_medium* m, double fs, double duration) {
  // make_passband (simulate.cpp:50-67)
  require(fs > 0.0 && duration > 0.0, "sampling rate and duration must be positive");
  require(fs >= m->min_fs_ratio * t->center_frequency,
          "sampling rate below the required multiple of the center frequency");
  RfsBand b;
  b.T = (int)std::llround(fs * duration);
  require(b.T >= 16, "duration too short for the sampling rate");
  b.df = fs / b.T;
  b.sigma = 0.5 * t->fractional_bandwidth * t->center_frequency / std::sqrt(2.0 * std::log(2.0));
  double span = std::sqrt(4.0 * std::log(10.0)) * b.sigma;
  int max_bin = (b.T - 1) / 2;
  b.j_lo = std::max(1, (int)std::ceil((t->center_frequency - span) / b.df));
  b.j_hi = std::min(max_bin, (int)std::floor((t->center_frequency + span) / b.df));
  require(b.j_lo <= b.j_hi, "no frequency bins fall inside the pulse passband");
  return b;
}

int rf_worker_count() {  // core/parallel.cpp:11-18
  if (const char* env = std::getenv("FQF_THREADS")) {
    int n = std::atoi(env);
    if (n >= 1) return n;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : (int)hw;
}

size_t rf_scratch_bytes(size_t vn, int nb, int n_elem) {  // simulate.cpp:212-216
  return (10 * vn + (size_t)nb + (size_t)nb * n_elem * 2 + (size_t)n_elem * 2) * sizeof(double);
}

// plan_layout (simulate.cpp:389-416): the reference engine's memory plan.
fqfg_rf_chunk_plan rf_plan_layout(const fqfg_transducer* t, size_t n_scat, const fqfg_medium* m,
                                  double fs, double duration, size_t budget, RfsBand* band_out) {
  require(n_scat > 0, "scatterer cloud is empty");
  RfsBand pb = rf_passband(t, m, fs, duration);
  size_t n_elem = (size_t)t->n_elements;
  size_t vn = n_elem * (size_t)t->subelements;
  fqfg_rf_chunk_plan plan{};
  plan.per_scatterer_bytes = (11 * vn + 2) * sizeof(double);
  int nb = std::min(64, pb.bins());
  size_t spec_bytes = (size_t)pb.bins() * n_elem * 2 * sizeof(double);
  size_t fftw_bytes = ((size_t)pb.T / 2 + 1) * 2 * sizeof(double) + (size_t)pb.T * sizeof(double);
  plan.fixed_bytes = 2 * spec_bytes + fftw_bytes + vn * 3 * sizeof(double) +
                     (size_t)rf_worker_count() * rf_scratch_bytes(vn, nb, (int)n_elem);
  require(budget >= plan.fixed_bytes + plan.per_scatterer_bytes,
          "memory budget cannot hold the fixed buffers plus one scatterer");
  size_t usable = budget - plan.fixed_bytes;
  plan.block_scatterers = std::min(n_scat, usable / plan.per_scatterer_bytes);
  plan.blocks = (int)((n_scat + plan.block_scatterers - 1) / plan.block_scatterers);
  if (band_out) *band_out = pb;
  return plan;
}

// check_inputs (simulate.cpp:349-387).
void rf_check_inputs(const double* pos, const double* refl, size_t n, const fqfg_transducer* t,
                     const double* delays, const double* apod, const fqfg_medium* m,
                     double duration) {
  rf_validate_transducer(t);
  require(n > 0 && pos, "scatterer cloud is empty");
  require(refl != nullptr, "cloud reflectivity count does not match positions");
  require(delays != nullptr, "transmit delays do not match element count");
  require(apod != nullptr, "transmit apodization does not match element count");
  require(m->c > 0.0, "sound speed must be positive");
  require(m->attenuation_db_cm_mhz >= 0.0, "attenuation must be nonnegative");
  double tau_max = 0.0;
  for (int e = 0; e < t->n_elements; ++e) {
    require(std::isfinite(delays[e]) && delays[e] >= 0.0,
            "transmit delays must be finite and nonnegative");
    tau_max = std::max(tau_max, delays[e]);
  }
  double xmin = t->xyz[0], xmax = xmin, ymin = t->xyz[1], ymax = ymin;
  for (int e = 0; e < t->n_elements; ++e) {
    xmin = std::min(xmin, t->xyz[3 * e]);
    xmax = std::max(xmax, t->xyz[3 * e]);
    ymin = std::min(ymin, t->xyz[3 * e + 1]);
    ymax = std::max(ymax, t->xyz[3 * e + 1]);
  }
  xmin -= t->half_width;
  xmax += t->half_width;
  double t_need = 0.0;
  for (size_t s = 0; s < n; ++s) {
    const double* p = pos + 3 * s;
    require(std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2]),
            "scatterer positions must be finite");
    double dx = std::max(std::abs(p[0] - xmin), std::abs(p[0] - xmax));
    double dy = std::max(std::abs(p[1] - ymin), std::abs(p[1] - ymax));
    double r_far = std::sqrt(dx * dx + dy * dy + p[2] * p[2]);
    t_need = std::max(t_need, tau_max + 2.0 * r_far / m->c);
  }
  for (size_t s = 0; s < n; ++s)
    require(std::isfinite(refl[s]), "scatterer reflectivities must be finite");
  require(duration >= t_need, "duration shorter than the maximum two-way travel time");
}

thread_local DevBuf tl_rfs_tx, tl_rfs_part, tl_rfs_spec, tl_rfs_tab, tl_rfs_in, tl_rfs_out;

// The GPU engine for one transmit event (device inputs, stream-ordered).
void run_rfsim(const double* d_pos, const double* d_refl, size_t n, const fqfg_transducer* t,
               const double* d_elem, const double* d_delays, const double* d_apod,
               const fqfg_medium* m, const RfsBand& pb, float* d_out32, double* d_out64,
               cudaStream_t st) {
  const int E = t->n_elements, nbins = pb.bins();
  // Segment table: 64-bin bands split at the 8-bin elevation knots.
  std::vector<RfsSeg> segs;
  for (int jb0 = pb.j_lo; jb0 <= pb.j_hi; jb0 += 64) {
    int nb = std::min(64, pb.j_hi - jb0 + 1);
    for (int sb0 = 0; sb0 < nb; sb0 += kRfsSeg) segs.push_back({jb0, nb, sb0, std::min(nb, sb0 + kRfsSeg)});
  }
  RfsParams p{};
  p.E = E;
  p.v = t->subelements;
  p.hw = t->half_width;
  p.c = m->c;
  p.df = pb.df;
  p.beta = m->attenuation_db_cm_mhz * (std::log(10.0) / 20.0) * 1e-4 * pb.df;
  p.elev = t->elevation_height > 0.0;
  p.wa = t->elevation_aperture_factor * t->elevation_height;
  p.inv_focus = p.elev ? 1.0 / t->elevation_focus : 0.0;
  p.core_w = t->elevation_core_weight;
  p.tail_w = t->elevation_tail_weight;
  p.j_lo = pb.j_lo;
  p.n_bins = nbins;
  p.n_seg = (int)segs.size();
  // Pulse weights (run_engine:484-489) and the exact twiddle table.
  std::vector<double> w(nbins);
  for (int j = pb.j_lo; j <= pb.j_hi; ++j) {
    double f = j * pb.df;
    double d = (f - t->center_frequency) / pb.sigma;
    w[j - pb.j_lo] = std::exp(-0.5 * d * d) / pb.T;
  }
  std::vector<double2> tw(pb.T);
  for (int k = 0; k < pb.T; ++k) {
    double th = 2.0 * 3.14159265358979323846 * (double)k / pb.T;
    tw[k] = make_double2(std::cos(th), std::sin(th));
  }
  const size_t tab_bytes = segs.size() * sizeof(RfsSeg) + 256 + nbins * sizeof(double) + 256 +
                           (size_t)pb.T * sizeof(double2);
  char* tab = static_cast<char*>(tl_rfs_tab.get(tab_bytes));
  RfsSeg* d_segs = reinterpret_cast<RfsSeg*>(tab);
  double* d_w = reinterpret_cast<double*>(tab + ((segs.size() * sizeof(RfsSeg) + 255) / 256) * 256);
  double2* d_tw = reinterpret_cast<double2*>(reinterpret_cast<char*>(d_w) +
                                             ((nbins * sizeof(double) + 255) / 256) * 256);
  CK(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(RfsSeg), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_w, w.data(), nbins * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_tw, tw.data(), pb.T * sizeof(double2), cudaMemcpyHostToDevice, st));
  int sms = 148, dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // TX(s, j): CTAs = segments x scatterer chunks (about 2 waves).
  const size_t want1 = std::max<size_t>(1, (size_t)(2 * sms) / segs.size() + 1);
  const size_t chunk1 = std::max<size_t>(1, (n + want1 - 1) / want1);
  const unsigned nchunk1 = (unsigned)((n + chunk1 - 1) / chunk1);
  double2* d_tx = static_cast<double2*>(tl_rfs_tx.get(n * nbins * sizeof(double2)));
  rfs_tx_kernel<<<dim3((unsigned)segs.size(), nchunk1), kRfsThreads, 0, st>>>(
      p, d_segs, d_pos, n, chunk1, d_elem, d_delays, d_apod, d_tx);
  CK_LAUNCH();
  // S(j, e): CTAs = segments x element tiles x scatterer chunks.
  const unsigned etiles = (unsigned)((E + kRfsThreads - 1) / kRfsThreads);
  size_t nchunk2 = std::max<size_t>(1, (size_t)(2 * sms) / (segs.size() * etiles) + 1);
  nchunk2 = std::min<size_t>({nchunk2, 64, n});
  const size_t chunk2 = (n + nchunk2 - 1) / nchunk2;
  nchunk2 = (n + chunk2 - 1) / chunk2;
  const size_t spec_n = (size_t)nbins * E;
  double2* d_part = static_cast<double2*>(tl_rfs_part.get(nchunk2 * spec_n * sizeof(double2)));
  rfs_spec_kernel<<<dim3((unsigned)segs.size(), etiles, (unsigned)nchunk2), kRfsThreads, 0, st>>>(
      p, d_segs, d_pos, d_refl, n, chunk2, d_elem, d_tx, d_part);
  CK_LAUNCH();
  double2* d_spec = static_cast<double2*>(tl_rfs_spec.get(spec_n * sizeof(double2)));
  rfs_reduce_kernel<<<(unsigned)((spec_n + 255) / 256), 256, 0, st>>>(d_part, (int)nchunk2,
                                                                      spec_n, d_spec);
  CK_LAUNCH();
  const size_t nout = (size_t)pb.T * E;
  rfs_idft_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>(d_spec, d_w, d_tw, pb.T, E,
                                                                  pb.j_lo, nbins, d_out64, d_out32);
  CK_LAUNCH();
}

}  // namespace

// ================================================================ C ABI ==

#pragma GCC visibility push(default)
extern "C" {

const char* fqfg_last_error(void) { return g_err.c_str(); }

int fqfg_version(void) { return 1; }

int fqfg_device_count(void) { return sm100_devices(); }

int fqfg_set_device(int device) {
  return guarded([&] {
    need_device();
    CK(cudaSetDevice(device));
  });
}

int fqfg_plan_chunks(size_t n_points, int n_angles, size_t budget, size_t* ranges,
                     size_t max_chunks, size_t* n_chunks) {
  return guarded([&] {
    std::vector<std::pair<size_t, size_t>> r;
    size_t k = plan_chunks(n_points, n_angles, budget, r);
    if (n_chunks) *n_chunks = k;
    if (ranges)
      for (size_t i = 0; i < std::min(k, max_chunks); ++i) {
        ranges[2 * i] = r[i].first;
        ranges[2 * i + 1] = r[i].second;
      }
  });
}

int fqfg_das_plan_create(const fqfg_rf_desc* rf, const fqfg_grid* grid, const fqfg_probe* probe,
                         const fqfg_bf* bf, fqfg_das_plan* out) {
  return guarded([&] {
    require(out != nullptr, "plan output pointer is null");
    need_device();
    auto* P = new fqfg_das_plan_s();
    CK(cudaGetDevice(&P->device));
    try {
      // The IQ of one frame pass may take up to 45 % of the device memory
      // (config D: 65 GB at 112 frames per pass on a 180 GB B200).
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      build_plan(rf, grid, probe, bf, *P, (size_t)(0.45 * (double)total_b));
    } catch (...) {
      free_plan(P);
      delete P;
      throw;
    }
    *out = P;
  });
}

int fqfg_das_plan_info_get(fqfg_das_plan P, fqfg_das_plan_info* info) {
  return guarded([&] {
    require(P && info, "null plan");
    info->n_points = (size_t)P->p.nx * P->p.ny * P->p.nz;
    info->frames_per_pass = P->p.fpass;
    info->n_passes = P->p.npass;
    info->work_bytes = P->stage_bytes + P->iq_bytes;
    info->active_pairs = P->active_pairs;
    info->tile[0] = P->TX;
    info->tile[1] = P->TY;
    info->tile[2] = P->TZ;
    info->shape[0] = P->J;
    info->shape[1] = P->VPW;
    info->shape[2] = P->NW;
    info->shape[3] = P->PW;
    info->mode = P->tc ? 2 : 0;
  });
}

void fqfg_das_plan_destroy(fqfg_das_plan P) {
  free_plan(P);
  delete P;
}

int fqfg_das_slab_samples(fqfg_das_plan P, int kb, int ke, int* t_begin, int* t_end) {
  return guarded([&] {
    require(P != nullptr && t_begin && t_end, "null argument");
    require(kb >= 0 && ke <= P->p.nz && kb < ke, "z-slab [%d, %d) outside the grid", kb, ke);
    int row_lo, row_hi;
    slab_rows(*P, kb, ke, row_lo, row_hi);
    const int mid = P->p.taps / 2;
    // RF samples feeding IQ samples [row_lo - 1, row_hi - 1] through the FIR.
    *t_begin = std::max(0, row_lo - 1 - mid);
    *t_end = std::min(P->p.T, std::max(*t_begin, row_hi + mid));
  });
}

int fqfg_copy_slices_h2d(void* d_dst, const void* h_src, size_t n, size_t slice, size_t off,
                         size_t bytes, void* stream) {
  return guarded([&] {
    require(off + bytes <= slice, "slice range outside the slice");
    if (n == 0 || bytes == 0) return;
    CK(cudaMemcpy2DAsync(static_cast<char*>(d_dst) + off, slice,
                         static_cast<const char*>(h_src) + off, slice, bytes, n,
                         cudaMemcpyHostToDevice, (cudaStream_t)stream));
  });
}

int fqfg_das_plan_set_timing(fqfg_das_plan P, int enable) {
  return guarded([&] {
    require(P != nullptr, "null plan");
    harvest_timing(*P);
    P->timing = enable != 0;
    P->acc_demod_ms = P->acc_das_ms = 0.0;
    P->acc_calls = 0;
  });
}

// Totals over the fqfg_das_dev calls since timing was enabled.
int fqfg_das_last_timing(fqfg_das_plan P, double* demod_ms, double* das_ms) {
  return guarded([&] {
    require(P != nullptr, "null plan");
    harvest_timing(*P);
    if (demod_ms) *demod_ms = P->acc_demod_ms;
    if (das_ms) *das_ms = P->acc_das_ms;
  });
}

uint64_t fqfg_launch_count(void) { return g_launches.load(); }

int fqfg_das_dev(fqfg_das_plan P, const float* d_rf, int kb, int ke, float* d_x, void* d_work,
                 uint64_t* d_counters, void* stream) {
  return guarded([&] {
    require(P != nullptr, "null plan");
    run_das(*P, d_rf, kb, ke, reinterpret_cast<float2*>(d_x), d_work,
            reinterpret_cast<unsigned long long*>(d_counters), (cudaStream_t)stream);
  });
}


size_t fqfg_gram_work_bytes(int F) { return gram_splits(F) * (size_t)F * F * sizeof(double2); }

int fqfg_gram_dev(const float* d_x, int F, size_t N, size_t v0, size_t v1, double* d_g,
                  void* d_work, void* stream) {
  return guarded([&] {
    require(F >= 1 && v0 <= v1 && v1 <= N, "bad Gram range");
    run_gram(reinterpret_cast<const float2*>(d_x), F, N, v0, v1, reinterpret_cast<double2*>(d_g),
             d_work, 0, (cudaStream_t)stream);
  });
}

size_t fqfg_gram_tc_work_bytes(int F) { return F >= 1 && F <= 1024 ? gram_tc_work_bytes(F) : 0; }

int fqfg_gram_tc_dev(const float* d_x, int F, size_t N, size_t v0, size_t v1, double* d_g,
                     void* d_work, void* stream) {
  return guarded([&] {
    require(F >= 1 && v0 <= v1 && v1 <= N, "bad Gram range");
    run_gram_tc(reinterpret_cast<const float2*>(d_x), F, N, v0, v1,
                reinterpret_cast<double2*>(d_g), d_work, 0, (cudaStream_t)stream);
  });
}

int fqfg_eig_dev(double* d_g, int F, double* d_w, double* d_v, void* stream) {
  return guarded([&] {
    void* vw = tl_eig.get(std::max(eig_work_bytes(F), (size_t)F * F * sizeof(double2)));
    run_eig(reinterpret_cast<double2*>(d_g), F, d_w, reinterpret_cast<double2*>(d_v), vw,
            (cudaStream_t)stream);
  });
}

int fqfg_eig_band_dev(double* d_g, int F, int lo, int hi, double* d_w, double* d_v,
                      void* stream) {
  return guarded([&] {
    check_filter(F, (size_t)F, lo, hi);
    void* vw = tl_eig.get(std::max(eig_work_bytes(F), (size_t)F * F * sizeof(double2)));
    run_eig_band(reinterpret_cast<double2*>(d_g), F, lo, hi, d_w, reinterpret_cast<double2*>(d_v),
                 vw, (cudaStream_t)stream);
  });
}

int fqfg_project_pd_dev(const float* d_x, int F, size_t N, size_t v0, size_t v1, const double* d_v,
                        int lo, int hi, float* d_y, double* d_pd, void* stream) {
  return guarded([&] {
    check_filter(F, N, lo, hi);
    void* scratch = tl_small.get(filter_scratch_bytes(F));
    run_project(reinterpret_cast<const float2*>(d_x), F, N, v0, v1,
                reinterpret_cast<const double2*>(d_v), lo, hi, reinterpret_cast<float2*>(d_y),
                d_pd, scratch, (cudaStream_t)stream);
  });
}

int fqfg_synth_rf_dev(float* d_rf, size_t n, uint64_t seed, void* stream) {
  return guarded([&] {
    synth_rf_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(d_rf, n, seed);
    CK_LAUNCH();
  });
}

int fqfg_rf_to_iq(const float* rf, int batch, int T, int E, double fs, const double* t0,
                  double fc, int taps, float* iq) {
  return guarded([&] {
    require(fc > 0.0, "demodulation frequency must be positive");
    require(fs > 2.0 * fc, "sampling rate must exceed twice the demodulation frequency");
    require(taps >= 3 && taps % 2 == 1, "low-pass tap count must be odd and at least 3");
    require(T >= 1 && E >= 1 && batch >= 1, "frame has no samples");
    require(taps <= 255, "low-pass tap count above 255 is not supported");
    need_device();
    cudaStream_t st = 0;
    size_t n = (size_t)batch * T * E;
    float* d_rf = static_cast<float*>(tl_rf.get(n * sizeof(float)));
    float2* d_iq = static_cast<float2*>(tl_x.get(n * sizeof(float2)));
    std::vector<double2> car = carrier_table(t0, batch, T, fc, fs);
    std::vector<double> h = lowpass(fc, fs, taps);
    std::vector<float> hf(h.begin(), h.end());
    char* small = static_cast<char*>(tl_small.get(car.size() * sizeof(double2) + 4096));
    double2* d_car = reinterpret_cast<double2*>(small);
    float* d_h = reinterpret_cast<float*>(small + car.size() * sizeof(double2));
    CK(cudaMemcpyAsync(d_rf, rf, n * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_car, car.data(), car.size() * sizeof(double2), cudaMemcpyHostToDevice,
                       st));
    CK(cudaMemcpyAsync(d_h, hf.data(), hf.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    const int rows = kDemodTB + taps - 1;
    size_t smem = (size_t)rows * 32 * sizeof(float2) + taps * sizeof(float);
    smem_attr((void*)demod_fir_kernel, smem);
    // Each frame of the batch is its own "angle" slot so it gets its own t0.
    dim3 g((T + kDemodTB - 1) / kDemodTB, (E + 31) / 32, batch);
    const RfSrc src{d_rf, (long long)batch * T * E, (long long)T * E, 0, T, 0};
    demod_fir_kernel<<<g, 256, smem, st>>>(src, d_iq, d_car, d_h, T, E, batch, taps);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(iq, d_iq, n * sizeof(float2), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_das(const fqfg_rf_desc* d, const float* rf, const fqfg_grid* grid,
             const fqfg_probe* probe, const fqfg_bf* bf, const fqfg_das_opts* opts_in,
             float* iq_out, fqfg_das_stats* stats) {
  return guarded([&] {
    fqfg_das_opts opts = opts_in ? *opts_in : fqfg_das_opts{100000000ull, 512000000ull, 1};
    check_rf(d, probe);
    check_grid(grid);
    size_t N = (size_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
    std::vector<std::pair<size_t, size_t>> ranges;
    size_t chunks = das_chunk_plan(N, d->n_angles, d->n_elements, bf ? bf->interp_order : 1, opts,
                                   ranges);
    need_device();
    fqfg_das_plan_s P;
    CK(cudaGetDevice(&P.device));
    struct Guard {
      fqfg_das_plan_s* p;
      ~Guard() { free_plan(p); }
    } guard{&P};
    build_plan(d, grid, probe, bf, P);
    const DasParams& p = P.p;
    cudaStream_t st = 0;
    size_t n_rf = (size_t)p.F * p.A * p.T * p.E;
    float* d_rf = static_cast<float*>(tl_rf.get(n_rf * sizeof(float)));
    float2* d_x = static_cast<float2*>(tl_x.get((size_t)p.F * N * sizeof(float2)));
    void* work = tl_work.get(P.stage_bytes + P.iq_bytes);
    unsigned long long* cnt = static_cast<unsigned long long*>(tl_cnt.get(64));
    CK(cudaMemsetAsync(cnt, 0, 16, st));
    CK(cudaMemcpyAsync(d_rf, rf, n_rf * sizeof(float), cudaMemcpyHostToDevice, st));
    run_das(P, d_rf, 0, p.nz, d_x, work, cnt, st);
    CK(cudaMemcpyAsync(iq_out, d_x, (size_t)p.F * N * sizeof(float2), cudaMemcpyDeviceToHost, st));
    if (stats) {
      unsigned* taps = static_cast<unsigned*>(tl_y.get(N * p.A * sizeof(unsigned)));
      CK(cudaMemsetAsync(cnt + 2, 0, 8, st));
      tap_stats_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(p, taps, cnt + 2);
      CK_LAUNCH();
      std::vector<unsigned> h_taps(N * p.A);
      unsigned long long oow = 0;
      CK(cudaMemcpyAsync(h_taps.data(), taps, h_taps.size() * sizeof(unsigned),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&oow, cnt + 2, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      fqfg_das_stats s{};
      s.chunks = chunks;
      s.matrix_builds = opts.cache_matrices ? chunks * p.A : chunks * p.A * (uint64_t)p.F;
      s.out_of_window = oow;
      size_t maxlen = 0, peak = 0;
      for (auto& r : ranges) {
        size_t len = r.second - r.first;
        maxlen = std::max(maxlen, len);
        size_t sum = 0;
        for (int a = 0; a < p.A; ++a) {
          size_t nnz = 0;
          for (size_t v = r.first; v < r.second; ++v) nnz += h_taps[v * p.A + a];
          size_t bytes = nnz * (16 + 4) + (len + 1) * 8;
          if (opts.cache_matrices)
            sum += bytes;
          else
            peak = std::max(peak, bytes);
        }
        if (opts.cache_matrices) peak = std::max(peak, sum);
      }
      s.matrix_bytes_peak = peak;
      s.accumulator_bytes_peak = 16ull * maxlen * p.A;
      *stats = s;
    }
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_svd_filter(const float* iq, int F, size_t N, int lo, int hi, float* filtered,
                    double* sigma, double* pd, double* corr) {
  return guarded([&] {
    check_filter(F, N, lo, hi);
    need_device();
    cudaStream_t st = 0;
    float2* d_x = static_cast<float2*>(tl_x.get((size_t)F * N * sizeof(float2)));
    float2* d_y = filtered ? static_cast<float2*>(tl_y.get((size_t)F * N * sizeof(float2))) : nullptr;
    double* d_pd = pd ? static_cast<double*>(tl_pd.get(N * sizeof(double))) : nullptr;
    CK(cudaMemcpyAsync(d_x, iq, (size_t)F * N * sizeof(float2), cudaMemcpyHostToDevice, st));
    run_filter(d_x, F, N, lo, hi, d_y, d_pd, sigma, st, corr);
    if (filtered)
      CK(cudaMemcpyAsync(filtered, d_y, (size_t)F * N * sizeof(float2), cudaMemcpyDeviceToHost, st));
    if (pd) CK(cudaMemcpyAsync(pd, d_pd, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_build_delay_matrix(const double* voxels, size_t n, double angle, double t0, double fs,
                            int T, const fqfg_probe* probe, const fqfg_bf* bf, uint64_t* row_ptr,
                            int32_t* col_idx, double* values, uint64_t* out_of_window,
                            int* padded_samples) {
  return guarded([&] {
    require(bf && bf->c > 0.0, "sound speed must be positive");
    require(bf->center_frequency > 0.0, "rotation frequency must be positive");
    require(bf->interp_order == 0 || bf->interp_order == 1,
            "interpolation order must be 0 (nearest) or 1 (linear)");
    require(fs > 0.0, "sampling rate must be positive");
    require(T >= 1, "recording must hold at least one sample");
    require(std::isfinite(angle) && std::fabs(angle) < kPi / 2.0,
            "steering angle must stay within the forward half-space");
    require(probe && probe->n_elements >= 1, "transducer has no elements");
    int E = probe->n_elements;
    require((size_t)T * E <= (size_t)std::numeric_limits<int32_t>::max(),
            "recording is too large for the column index width");
    for (size_t v = 0; v < 3 * n; ++v)
      require(std::isfinite(voxels[v]), "voxel position must be finite");
    require(row_ptr != nullptr, "row_ptr is required");
    need_device();
    cudaStream_t st = 0;
    DmParams q{};
    q.sina = std::sin(angle);
    q.cosa = std::cos(angle);
    q.ref = std::numeric_limits<double>::infinity();
    for (int e = 0; e < E; ++e) q.ref = std::min(q.ref, probe->xyz[3 * e] * q.sina);
    q.t0 = t0;
    q.fs = fs;
    q.c = bf->c;
    q.omega = 2.0 * kPi * bf->center_frequency;
    q.fnum = bf->f_number;
    q.E = E;
    q.T = T;
    q.interp = bf->interp_order;
    size_t nn = std::max<size_t>(n, 1);
    char* buf = static_cast<char*>(tl_small.get(3 * nn * sizeof(double) + 3 * (size_t)E * sizeof(double) +
                                                (nn + 1) * 8 + 64));
    double* d_vox = reinterpret_cast<double*>(buf);
    double* d_el = d_vox + 3 * nn;
    unsigned long long* d_len = reinterpret_cast<unsigned long long*>(d_el + 3 * E);
    unsigned long long* d_oow = d_len + nn;
    long long* d_last = reinterpret_cast<long long*>(d_oow + 1);
    q.elem = d_el;
    if (n) CK(cudaMemcpyAsync(d_vox, voxels, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_el, probe->xyz, 3 * (size_t)E * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_oow, 0, 8, st));
    long long init_last = T - 1;
    CK(cudaMemcpyAsync(d_last, &init_last, 8, cudaMemcpyHostToDevice, st));
    if (n) {
      dm_count_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(q, d_vox, n, d_len, d_oow,
                                                                     d_last);
      CK_LAUNCH();
    }
    std::vector<unsigned long long> len(n);
    unsigned long long oow = 0;
    long long last = 0;
    if (n) CK(cudaMemcpyAsync(len.data(), d_len, n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&oow, d_oow, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last, d_last, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    row_ptr[0] = 0;
    for (size_t v = 0; v < n; ++v) row_ptr[v + 1] = row_ptr[v] + len[v];
    if (out_of_window) *out_of_window = oow;
    if (padded_samples) {
      long long cap = std::numeric_limits<int32_t>::max() / E - 1;
      *padded_samples = (int)std::min(last, cap) + 1;
    }
    if (!col_idx || !values || n == 0) return;
    size_t nnz = row_ptr[n];
    size_t rp_bytes = ((n + 1) * 8 + 255) / 256 * 256;  // keep double2 16-byte aligned
    char* out = static_cast<char*>(tl_y.get(rp_bytes + nnz * (4 + 16) + 64));
    unsigned long long* d_rp = reinterpret_cast<unsigned long long*>(out);
    double2* d_val = reinterpret_cast<double2*>(out + rp_bytes);
    int* d_col = reinterpret_cast<int*>(d_val + nnz);
    CK(cudaMemcpyAsync(d_rp, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, st));
    dm_fill_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(q, d_vox, n, d_rp, d_col, d_val);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(col_idx, d_col, nnz * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(values, d_val, nnz * 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_apply_delay_matrix(size_t rows, const uint64_t* row_ptr, const int32_t* col_idx,
                            const double* values, const double* iq, size_t n_iq, double* out) {
  return guarded([&] {
    need_device();
    size_t nnz = row_ptr[rows];
    for (size_t i = 0; i < nnz; ++i)
      require(col_idx[i] >= 0 && (size_t)col_idx[i] < n_iq,
              "delay-matrix column %d outside the frame", (int)col_idx[i]);
    cudaStream_t st = 0;
    size_t rp_bytes = ((rows + 1) * 8 + 255) / 256 * 256;  // keep double2 16-byte aligned
    char* buf = static_cast<char*>(
        tl_y.get(rp_bytes + nnz * 20 + n_iq * 16 + std::max<size_t>(rows, 1) * 16 + 256));
    unsigned long long* d_rp = reinterpret_cast<unsigned long long*>(buf);
    double2* d_val = reinterpret_cast<double2*>(buf + rp_bytes);
    double2* d_iq = d_val + nnz;
    double2* d_out = d_iq + n_iq;
    int* d_col = reinterpret_cast<int*>(d_out + std::max<size_t>(rows, 1));
    CK(cudaMemcpyAsync(d_rp, row_ptr, (rows + 1) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_val, values, nnz * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_iq, iq, n_iq * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_col, col_idx, nnz * 4, cudaMemcpyHostToDevice, st));
    if (rows) {
      dm_apply_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(rows, d_rp, d_col, d_val,
                                                                       d_iq, d_out);
      CK_LAUNCH();
      CK(cudaMemcpyAsync(out, d_out, rows * 16, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_power_doppler(const float* iq, int F, size_t N, double* pd) {
  return guarded([&] {
    require(F >= 1, "power_doppler needs at least one frame");
    require(N > 0, "power_doppler needs a nonempty grid");
    need_device();
    cudaStream_t st = 0;
    float2* d_x = static_cast<float2*>(tl_x.get((size_t)F * N * sizeof(float2)));
    double* d_pd = static_cast<double*>(tl_pd.get(N * sizeof(double)));
    CK(cudaMemcpyAsync(d_x, iq, (size_t)F * N * sizeof(float2), cudaMemcpyHostToDevice, st));
    power_doppler_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(d_x, F, N, 0, N, d_pd);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(pd, d_pd, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}


// ------------------------------------------------ display and scoring --

int fqfg_render_db(const double* vol, const int* dims, double dr_db, int power, double* out) {
  return guarded([&] {
    require(vol && dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0,
            "render_db needs a nonempty volume");
    require(dr_db > 0.0, "dynamic range must be positive, got %g", dr_db);
    need_device();
    const size_t n = dims_points(dims);
    cudaStream_t st = 0;
    double* d_in = static_cast<double*>(tl_disp_a.get(n * sizeof(double)));
    double* d_out = static_cast<double*>(tl_pd.get(n * sizeof(double)));
    CK(cudaMemcpyAsync(d_in, vol, n * sizeof(double), cudaMemcpyHostToDevice, st));
    run_render_db(d_in, n, dr_db, power != 0, d_out, st);
    CK(cudaMemcpyAsync(out, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_render_db_dev(const double* d_vol, size_t n, double dr_db, int power, double* d_out,
                       void* stream) {
  return guarded([&] {
    require(n > 0, "render_db needs a nonempty volume");
    require(dr_db > 0.0, "dynamic range must be positive, got %g", dr_db);
    need_device();
    run_render_db(d_vol, n, dr_db, power != 0, d_out, (cudaStream_t)stream);
  });
}

int fqfg_bmode(const double* iq, const int* dims, double dr_db, double* out) {
  return guarded([&] {
    require(iq && dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0,
            "bmode needs an IQ volume matching its grid");
    require(dr_db > 0.0, "dynamic range must be positive, got %g", dr_db);
    need_device();
    const size_t n = dims_points(dims);
    cudaStream_t st = 0;
    double2* d_iq = static_cast<double2*>(tl_disp_a.get(n * sizeof(double2)));
    double* d_env = static_cast<double*>(tl_disp_b.get(n * sizeof(double)));
    double* d_out = static_cast<double*>(tl_pd.get(n * sizeof(double)));
    CK(cudaMemcpyAsync(d_iq, iq, n * sizeof(double2), cudaMemcpyHostToDevice, st));
    cabs_kernel<<<disp_blocks(n), kDispThreads, 0, st>>>(d_iq, n, d_env);
    CK_LAUNCH();
    run_render_db(d_env, n, dr_db, false, d_out, st);
    CK(cudaMemcpyAsync(out, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_mip(const double* vol, const int* dims, int axis, double* out) {
  return guarded([&] {
    require(axis >= 0 && axis < 3, "mip axis must be 0, 1, or 2, got %d", axis);
    require(vol && dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0,
            "mip needs a nonempty volume");
    need_device();
    const size_t n = dims_points(dims);
    const size_t m = n / (size_t)dims[axis];
    cudaStream_t st = 0;
    double* d_in = static_cast<double*>(tl_disp_a.get(n * sizeof(double)));
    double* d_out = static_cast<double*>(tl_disp_b.get(m * sizeof(double)));
    CK(cudaMemcpyAsync(d_in, vol, n * sizeof(double), cudaMemcpyHostToDevice, st));
    mip_kernel<<<disp_blocks(m), kDispThreads, 0, st>>>(d_in, dims[0], dims[1], dims[2], axis,
                                                         d_out);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(out, d_out, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_ground_truth_pd(const double* xyz, const int* counts, int n_frames,
                         const fqfg_grid* grid, double sigma_voxels, double* out) {
  return guarded([&] {
    require(n_frames >= 1 && counts, "ground_truth_pd needs at least one frame");
    require(grid && grid->dims[0] > 0 && grid->dims[1] > 0 && grid->dims[2] > 0,
            "ground_truth_pd needs a nonempty grid");
    require(sigma_voxels > 0.0, "kernel sigma must be positive, got %g", sigma_voxels);
    size_t ns = 0;
    for (int f = 0; f < n_frames; ++f) {
      require(counts[f] >= 0, "negative scatterer count");
      ns += (size_t)counts[f];
    }
    for (size_t s = 0; s < ns; ++s) {
      for (int a = 0; a < 3; ++a) {
        const double u = (xyz[3 * s + a] - grid->origin[a]) / grid->spacing[a];
        require(std::isfinite(u), "scatterer positions must be finite");
      }
    }
    need_device();
    const size_t n = (size_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
    cudaStream_t st = 0;
    double* d_xyz = static_cast<double*>(tl_disp_a.get(std::max<size_t>(ns, 1) * 3 * sizeof(double)));
    double* d_out = static_cast<double*>(tl_pd.get(n * sizeof(double)));
    if (ns) CK(cudaMemcpyAsync(d_xyz, xyz, ns * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_out, 0, n * sizeof(double), st));
    SplatGrid g;
    g.nx = grid->dims[0], g.ny = grid->dims[1], g.nz = grid->dims[2];
    g.ox = grid->origin[0], g.oy = grid->origin[1], g.oz = grid->origin[2];
    g.sx = grid->spacing[0], g.sy = grid->spacing[1], g.sz = grid->spacing[2];
    g.reach = 3.0 * sigma_voxels;
    g.reach2 = g.reach * g.reach;
    g.inv_two_sigma2 = 1.0 / (2.0 * sigma_voxels * sigma_voxels);
    // every contribution is <= 1, so a voxel sum is <= ns: 62 - ceil(log2(ns
    // + 1)) fraction bits cannot overflow
    const int bits = std::min(52, 62 - (int)std::ceil(std::log2((double)ns + 1.0)));
    g.fx = std::ldexp(1.0, bits);
    g.inv_fx = std::ldexp(1.0, -bits);
    if (ns) {
      splat_kernel<<<disp_blocks(ns), kDispThreads, 0, st>>>(d_xyz, ns, g, d_out);
      CK_LAUNCH();
      fixed_to_double_kernel<<<disp_blocks(n), kDispThreads, 0, st>>>(d_out, n, g.inv_fx);
      CK_LAUNCH();
    }
    auto* peak = static_cast<unsigned long long*>(tl_disp_pk.get(sizeof(unsigned long long)));
    CK(cudaMemsetAsync(peak, 0, sizeof(unsigned long long), st));
    peak_abs_kernel<<<std::min(disp_blocks(n), 1184u), kDispThreads, 0, st>>>(d_out, n, peak);
    CK_LAUNCH();
    scale_kernel<<<disp_blocks(n), kDispThreads, 0, st>>>(d_out, n, peak);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(out, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fqfg_metrics(const double* test, const double* reference, const int* dims,
                 double* mse_psnr_ssim) {
  return guarded([&] {
    require(test && reference && dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0,
            "metrics needs nonempty images");
    need_device();
    const size_t n = dims_points(dims);
    cudaStream_t st = 0;
    double* d_a = static_cast<double*>(tl_disp_a.get(2 * n * sizeof(double)));
    CK(cudaMemcpyAsync(d_a, test, n * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_a + n, reference, n * sizeof(double), cudaMemcpyHostToDevice, st));
    run_metrics(d_a, d_a + n, dims, mse_psnr_ssim, st);
  });
}

int fqfg_metrics_dev(const double* d_test, const double* d_reference, const int* dims,
                     double* mse_psnr_ssim, void* stream) {
  return guarded([&] {
    require(d_test && d_reference && dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0,
            "metrics needs nonempty images");
    need_device();
    run_metrics(d_test, d_reference, dims, mse_psnr_ssim, (cudaStream_t)stream);
  });
}

// ------------------------------------------------------- RF synthesis --

int fqfg_plan_rf_chunks(const fqfg_transducer* t, size_t n_scatterers, const fqfg_medium* m,
                        double sampling_rate, double duration, size_t budget,
                        fqfg_rf_chunk_plan* out) {
  return guarded([&] {
    rf_validate_transducer(t);
    require(m != nullptr, "medium parameters missing");
    require(n_scatterers > 0, "scatterer cloud is empty");
    *out = rf_plan_layout(t, n_scatterers, m, sampling_rate, duration, budget, nullptr);
  });
}

int fqfg_simulate_rf(const double* positions, const double* reflectivity, size_t n,
                     const fqfg_transducer* t, const double* tx_delays, const double* tx_apod,
                     const fqfg_medium* m, double fs, double duration, int chunked, size_t budget,
                     double* rf_out, int* n_samples, fqfg_rfsim_stats* stats) {
  return guarded([&] {
    rf_validate_transducer(t);
    require(m != nullptr, "medium parameters missing");
    require(n > 0, "scatterer cloud is empty");
    const size_t bud = chunked ? (budget ? budget : m->scatterer_memory_budget)
                               : m->scatterer_memory_budget;
    RfsBand pb;
    fqfg_rf_chunk_plan plan = rf_plan_layout(t, n, m, fs, duration, bud, &pb);
    if (!chunked)
      require(plan.blocks == 1,
              "pair geometry exceeds the scatterer memory budget; use simulate_rf_chunked");
    rf_check_inputs(positions, reflectivity, n, t, tx_delays, tx_apod, m, duration);
    need_device();
    cudaStream_t st = 0;
    const int E = t->n_elements;
    const size_t in_bytes = (3 * n + n + 3 * (size_t)E + 2 * (size_t)E) * sizeof(double);
    double* d_in = static_cast<double*>(tl_rfs_in.get(in_bytes));
    double *d_pos = d_in, *d_refl = d_pos + 3 * n, *d_el = d_refl + n, *d_del = d_el + 3 * E,
           *d_apod = d_del + E;
    CK(cudaMemcpyAsync(d_pos, positions, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_refl, reflectivity, n * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_el, t->xyz, 3 * (size_t)E * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_del, tx_delays, E * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_apod, tx_apod, E * sizeof(double), cudaMemcpyHostToDevice, st));
    const size_t nout = (size_t)pb.T * E;
    double* d_out = static_cast<double*>(tl_rfs_out.get(nout * sizeof(double)));
    run_rfsim(d_pos, d_refl, n, t, d_el, d_del, d_apod, m, pb, nullptr, d_out, st);
    CK(cudaMemcpyAsync(rf_out, d_out, nout * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (size_t i = 0; i < nout; ++i)
      require(std::isfinite(rf_out[i]), "non-finite output sample: simulation unstable");
    if (n_samples) *n_samples = pb.T;
    if (stats) {
      const size_t vn = (size_t)E * t->subelements;
      const size_t geo = (11 * plan.block_scatterers * vn + 2 * plan.block_scatterers) * sizeof(double);
      const size_t fftw = ((size_t)pb.T / 2 + 1) * 2 * sizeof(double) + (size_t)pb.T * sizeof(double);
      stats->blocks = plan.blocks;
      stats->frequencies = pb.bins();
      stats->peak_tracked_bytes = plan.fixed_bytes - fftw + std::max(geo, fftw);
      stats->pair_bin_products = (uint64_t)n * vn * (uint64_t)pb.bins();
    }
  });
}

int fqfg_simulate_rf_dev(const double* d_positions, const double* d_reflectivity, size_t n,
                         const fqfg_transducer* t, const double* d_elements,
                         const double* d_tx_delays, const double* d_tx_apod, const fqfg_medium* m,
                         double fs, double duration, float* d_rf32, double* d_rf64, void* stream) {
  return guarded([&] {
    rf_validate_transducer(t);
    require(m != nullptr && m->c > 0.0, "sound speed must be positive");
    require(n > 0, "scatterer cloud is empty");
    need_device();
    RfsBand pb = rf_passband(t, m, fs, duration);
    run_rfsim(d_positions, d_reflectivity, n, t, d_elements, d_tx_delays, d_tx_apod, m, pb, d_rf32,
              d_rf64, (cudaStream_t)stream);
  });
}

}  // extern "C"
#pragma GCC visibility pop

#include "recon.cu"

