// fqf_dropin.cpp -- the reference's C++ reconstruction API, implemented over the
// B200 C ABI (include/fqfgpu.h).
//
// Compiled against the reference's own headers (-I <reference>/proj/include),
// so every signature below is the reference's by construction; no header is
// copied.  It replaces these reference translation units in a libfqf build:
//
//   proj/src/beamform/iq.cpp      rf_to_iq
//   proj/src/beamform/das.cpp     plan_chunks, build_delay_matrix, apply_delay_matrix,
//                                 das_reconstruct, assemble_frames, write/read_iq_volume
//   proj/src/post/svd.cpp         svd_filter
//   proj/src/post/render.cpp      power_doppler, render_db, bmode, mip, ground_truth_pd
//                                 (write_pgm stays)
//   proj/src/post/metrics.cpp     metrics (metrics_csv / metrics_json stay)
//
// Every compute step runs in libfqfgpu.so on the GPU; this file validates
// (same require() messages), marshals double <-> f32/complex64 and performs
// the reference's file side effects.  A nonzero C-ABI status becomes
// fqf::Error(fqfg_last_error()).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <filesystem>
#include <limits>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "fqf/beamform/das.hpp"
#include "fqf/beamform/iq.hpp"
#include "fqf/core/container.hpp"
#include "fqf/core/error.hpp"
#include "fqf/core/grid.hpp"
#include "fqf/post/metrics.hpp"
#include "fqf/post/render.hpp"
#include "fqf/post/svd.hpp"
#include "fqfgpu.h"

namespace fqf {
namespace {

constexpr double kPi = 3.14159265358979323846;

void ok(int rc) {
  if (rc != FQFG_OK) throw Error(fqfg_last_error());
}

std::string fmt17(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

void parse3(const std::string& s, double out[3]) {
  std::istringstream is(s);
  is >> out[0] >> out[1] >> out[2];
  require(!is.fail(), "bad 3-vector header value '", s, "'");
}

fqfg_bf c_bf(const beamform::BeamformParams& bp) {
  return fqfg_bf{bp.c, bp.center_frequency, bp.f_number, bp.interp_order, bp.lowpass_taps};
}

std::vector<double> flat_elements(const rf::Transducer& td) {
  std::vector<double> v;
  v.reserve(3 * td.elements.size());
  for (const Vec3& e : td.elements) {
    v.push_back(e.x);
    v.push_back(e.y);
    v.push_back(e.z);
  }
  return v;
}

std::vector<std::pair<std::size_t, std::size_t>> ranges_of(std::size_t n, std::size_t k) {
  std::vector<std::pair<std::size_t, std::size_t>> r;
  std::size_t base = n / k, rem = n % k, at = 0;
  for (std::size_t i = 0; i < k; ++i) {
    std::size_t len = base + (i < rem ? 1 : 0);
    r.emplace_back(at, at + len);
    at += len;
  }
  return r;
}

}  // namespace

namespace beamform {

// ----------------------------------------------------------------- iq.cpp --

IqFrame rf_to_iq(const rf::RfFrame& rfm, double f_c, int lowpass_taps) {
  require(f_c > 0.0, "demodulation frequency must be positive");
  require(rfm.sampling_rate > 2.0 * f_c,
          "sampling rate must exceed twice the demodulation frequency");
  require(lowpass_taps >= 3 && lowpass_taps % 2 == 1,
          "low-pass tap count must be odd and at least 3");
  require(rfm.n_samples >= 1 && rfm.n_elements >= 1, "frame has no samples");
  require(rfm.samples.size() ==
              static_cast<std::size_t>(rfm.n_samples) * static_cast<std::size_t>(rfm.n_elements),
          "frame buffer does not match its declared shape");
  std::vector<float> rf(rfm.samples.begin(), rfm.samples.end());
  std::vector<std::complex<float>> iq(rf.size());
  double t0 = rfm.t0;
  ok(fqfg_rf_to_iq(rf.data(), 1, rfm.n_samples, rfm.n_elements, rfm.sampling_rate, &t0, f_c,
                   lowpass_taps, reinterpret_cast<float*>(iq.data())));
  IqFrame out;
  out.n_samples = rfm.n_samples;
  out.n_elements = rfm.n_elements;
  out.sampling_rate = rfm.sampling_rate;
  out.t0 = rfm.t0;
  out.center_frequency = f_c;
  out.samples.assign(iq.begin(), iq.end());
  return out;
}

// ---------------------------------------------------------------- das.cpp --

std::size_t ChunkPlan::max_chunk_points() const {
  std::size_t m = 0;
  for (const auto& r : ranges) m = std::max(m, r.second - r.first);
  return m;
}

ChunkPlan plan_chunks(std::size_t n_points, int n_angles, std::size_t budget_bytes) {
  std::size_t k = 0;
  ok(fqfg_plan_chunks(n_points, n_angles, budget_bytes, nullptr, 0, &k));
  std::vector<std::size_t> r(2 * k);
  ok(fqfg_plan_chunks(n_points, n_angles, budget_bytes, r.data(), k, &k));
  ChunkPlan p;
  p.n_points = n_points;
  p.n_angles = n_angles;
  p.budget_bytes = budget_bytes;
  p.n_chunks = static_cast<int>(k);
  for (std::size_t i = 0; i < k; ++i) p.ranges.emplace_back(r[2 * i], r[2 * i + 1]);
  return p;
}

std::size_t DelayMatrix::bytes() const {
  return values.size() * sizeof(std::complex<double>) + col_idx.size() * sizeof(std::int32_t) +
         row_ptr.size() * sizeof(std::size_t);
}

DelayMatrix build_delay_matrix(std::span<const Vec3> voxels, const rf::TxEvent& tx,
                               const rf::Transducer& td, const BeamformParams& bp,
                               double sampling_rate, double t0, int n_time_samples) {
  std::vector<double> el = flat_elements(td);
  fqfg_probe probe{td.n_elements(), el.data()};
  fqfg_bf bf = c_bf(bp);
  std::vector<double> vox;
  vox.reserve(3 * voxels.size());
  for (const Vec3& p : voxels) {
    vox.push_back(p.x);
    vox.push_back(p.y);
    vox.push_back(p.z);
  }
  std::vector<std::uint64_t> rp(voxels.size() + 1);
  std::uint64_t oow = 0;
  int padded = 0;
  ok(fqfg_build_delay_matrix(vox.data(), voxels.size(), tx.angle, t0, sampling_rate,
                             n_time_samples, &probe, &bf, rp.data(), nullptr, nullptr, &oow,
                             &padded));
  DelayMatrix m;
  m.rows = voxels.size();
  m.n_elements = td.n_elements();
  m.recorded_samples = n_time_samples;
  m.padded_samples = padded;
  m.angle = tx.angle;
  m.interp_order = bp.interp_order;
  m.out_of_window = oow;
  std::size_t nnz = rp.back();
  m.col_idx.resize(nnz);
  m.values.resize(nnz);
  if (nnz)
    ok(fqfg_build_delay_matrix(vox.data(), voxels.size(), tx.angle, t0, sampling_rate,
                               n_time_samples, &probe, &bf, rp.data(), m.col_idx.data(),
                               reinterpret_cast<double*>(m.values.data()), &oow, &padded));
  m.row_ptr.assign(rp.begin(), rp.end());
  return m;
}

void apply_delay_matrix(const DelayMatrix& m, const IqFrame& iq, std::complex<double>* out) {
  require(iq.n_elements == m.n_elements, "frame element count does not match the matrix");
  require(iq.n_samples == m.recorded_samples, "frame length does not match the matrix");
  std::vector<std::uint64_t> rp(m.row_ptr.begin(), m.row_ptr.end());
  ok(fqfg_apply_delay_matrix(m.rows, rp.data(), m.col_idx.data(),
                             reinterpret_cast<const double*>(m.values.data()),
                             reinterpret_cast<const double*>(iq.samples.data()), iq.samples.size(),
                             reinterpret_cast<double*>(out)));
}

namespace {

void check_grid(const GridSpec& grid) {
  require(grid.dims[0] >= 1 && grid.dims[1] >= 1 && grid.dims[2] >= 1,
          "reconstruction grid dims must be positive");
  require(grid.spacing.x > 0 && grid.spacing.y > 0 && grid.spacing.z > 0,
          "reconstruction grid spacing must be positive");
  require(std::isfinite(grid.origin.x) && std::isfinite(grid.origin.y) &&
              std::isfinite(grid.origin.z),
          "reconstruction grid origin must be finite");
}

std::string scratch_dir() {
  auto base = std::filesystem::temp_directory_path();
  std::random_device rd;
  for (int attempt = 0; attempt < 16; ++attempt) {
    std::ostringstream os;
    os << "fqf_das_" << std::hex << rd() << rd();
    auto dir = base / os.str();
    std::error_code ec;
    if (std::filesystem::create_directory(dir, ec)) return dir.string();
  }
  fail("could not create a scratch directory under ", base.string());
}

// das_reconstruct's chunking (das.cpp:256-274), for the file layout and stats.
std::vector<std::pair<std::size_t, std::size_t>> das_ranges(std::size_t n, int A, int E,
                                                            const BeamformParams& bp,
                                                            const DasOptions& o) {
  ChunkPlan plan = plan_chunks(n, A, o.memory_budget_bytes);
  std::size_t resident = o.cache_matrices ? static_cast<std::size_t>(A) : 1;
  std::size_t taps = bp.interp_order == 0 ? 1 : 2;
  std::size_t per_voxel = taps * static_cast<std::size_t>(E) * 20 + 8;
  std::size_t maxlen = plan.max_chunk_points();
  if (resident * (maxlen * taps * E * 20 + (maxlen + 1) * 8) > o.matrix_budget_bytes) {
    std::size_t per_chunk = o.matrix_budget_bytes / resident;
    std::size_t cap = per_chunk > 8 ? (per_chunk - 8) / per_voxel : 0;
    require(cap >= 1, "delay-matrix budget cannot hold one voxel row");
    std::size_t k = std::max<std::size_t>(plan.n_chunks, (n + cap - 1) / cap);
    return ranges_of(n, k);
  }
  return plan.ranges;
}

}  // namespace

std::vector<IqVolume> das_reconstruct(const std::vector<std::vector<rf::RfFrame>>& frames,
                                      const GridSpec& grid, const rf::Transducer& td,
                                      const BeamformParams& bp, const DasOptions& opts,
                                      DasStats* stats) {
  require(!frames.empty(), "no frames to reconstruct");
  const int F = static_cast<int>(frames.size());
  const int A = static_cast<int>(frames[0].size());
  require(A >= 1, "frames carry no transmits");
  rf::validate_transducer(td);
  check_grid(grid);
  const int E = td.n_elements();
  const rf::RfFrame& first = frames[0][0];
  const double fs = first.sampling_rate;
  const int T = first.n_samples;
  require(fs > 0.0 && T >= 1, "frames are empty");
  for (int f = 0; f < F; ++f) {
    require(static_cast<int>(frames[f].size()) == A, "transmit count differs between frames");
    for (int a = 0; a < A; ++a) {
      const rf::RfFrame& fr = frames[f][a];
      require(fr.sampling_rate == fs, "sampling rate differs between frames");
      require(fr.n_samples == T, "sample count differs between frames");
      require(fr.n_elements == E, "element count does not match the transducer");
      require(fr.samples.size() == static_cast<std::size_t>(T) * E,
              "frame buffer does not match its declared shape");
      require(fr.tx.angle == frames[0][a].tx.angle,
              "transmit angle differs between frames at the same slot");
      require(fr.t0 == frames[0][a].t0, "start time differs between frames at the same slot");
    }
  }
  const std::size_t N = grid.num_points();
  std::vector<float> rf(static_cast<std::size_t>(F) * A * T * E);
  std::vector<double> t0(A), angles(A);
  for (int a = 0; a < A; ++a) {
    t0[a] = frames[0][a].t0;
    angles[a] = frames[0][a].tx.angle;
  }
  for (int f = 0; f < F; ++f)
    for (int a = 0; a < A; ++a)
      std::copy(frames[f][a].samples.begin(), frames[f][a].samples.end(),
                rf.begin() + (static_cast<std::size_t>(f) * A + a) * T * E);
  std::vector<double> el = flat_elements(td);
  fqfg_rf_desc desc{F, A, T, E, fs, t0.data(), angles.data()};
  fqfg_grid g{{grid.dims[0], grid.dims[1], grid.dims[2]},
              {grid.spacing.x, grid.spacing.y, grid.spacing.z},
              {grid.origin.x, grid.origin.y, grid.origin.z}};
  fqfg_probe probe{E, el.data()};
  fqfg_bf bf = c_bf(bp);
  fqfg_das_opts o{opts.memory_budget_bytes, opts.matrix_budget_bytes, opts.cache_matrices ? 1 : 0};
  std::vector<std::complex<float>> iq(static_cast<std::size_t>(F) * N);
  fqfg_das_stats st{};
  ok(fqfg_das(&desc, rf.data(), &g, &probe, &bf, &o, reinterpret_cast<float*>(iq.data()), &st));

  std::vector<IqVolume> volumes(F);
  for (int f = 0; f < F; ++f) {
    volumes[f].grid = grid;
    volumes[f].frame_index = f;
    volumes[f].n_angles = A;
    volumes[f].values.assign(iq.begin() + static_cast<std::size_t>(f) * N,
                             iq.begin() + static_cast<std::size_t>(f + 1) * N);
  }

  // File side effects (das.cpp:280-352): the GPU keeps the ensemble resident,
  // so chunk stripes exist only when the caller asks to keep them.
  if (opts.keep_chunk_files || opts.write_frames) {
    const bool auto_dir = opts.work_dir.empty();
    const std::string dir = auto_dir ? scratch_dir() : opts.work_dir;
    if (!auto_dir) std::filesystem::create_directories(dir);
    if (opts.keep_chunk_files) {
      auto ranges = das_ranges(N, A, E, bp, opts);
      for (std::size_t ci = 0; ci < ranges.size(); ++ci) {
        auto [b, e] = ranges[ci];
        std::vector<std::complex<double>> stripe;
        stripe.reserve((e - b) * F);
        for (int f = 0; f < F; ++f)
          stripe.insert(stripe.end(), volumes[f].values.begin() + b,
                        volumes[f].values.begin() + e);
        ContainerHeader h{{"kind", "iq_chunk"},
                          {"chunk", std::to_string(ci + 1)},
                          {"begin", std::to_string(b)},
                          {"end", std::to_string(e)},
                          {"frames", std::to_string(F)},
                          {"n_angles", std::to_string(A)}};
        write_container(dir + "/IQ_CHUNK_" + std::to_string(ci + 1) + ".fqf", h,
                        make_payload(std::span<const std::complex<double>>(stripe)));
      }
    }
    if (opts.write_frames)
      for (int f = 0; f < F; ++f)
        write_iq_volume(dir + "/Frame_" + std::to_string(f + 1) + ".fqf", volumes[f]);
  }
  if (stats) {
    stats->chunks = static_cast<int>(st.chunks);
    stats->matrix_builds = static_cast<int>(st.matrix_builds);
    stats->out_of_window = st.out_of_window;
    stats->matrix_bytes_peak = st.matrix_bytes_peak;
    stats->accumulator_bytes_peak = st.accumulator_bytes_peak;
  }
  return volumes;
}

std::vector<IqVolume> assemble_frames(const std::string& work_dir, const ChunkPlan& plan,
                                      const GridSpec& grid, int n_frames) {
  require(n_frames >= 1, "no frames to assemble");
  require(plan.n_points == grid.num_points(), "chunk plan does not match the grid");
  require(plan.n_chunks == static_cast<int>(plan.ranges.size()), "chunk plan is inconsistent");
  std::vector<IqVolume> out(n_frames);
  for (int f = 0; f < n_frames; ++f) {
    out[f].grid = grid;
    out[f].frame_index = f;
    out[f].values.assign(plan.n_points, {0.0, 0.0});
  }
  for (int ci = 0; ci < plan.n_chunks; ++ci) {
    const auto [b, e] = plan.ranges[ci];
    const std::string path = work_dir + "/IQ_CHUNK_" + std::to_string(ci + 1) + ".fqf";
    require(std::filesystem::exists(path), "missing chunk file ", path);
    auto [h, payload] = read_container(path);
    require(header_value(h, "kind") == "iq_chunk", path, ": not a chunk file");
    require(std::stoi(header_value(h, "chunk")) == ci + 1, path, ": chunk index mismatch");
    require(std::stoull(header_value(h, "begin")) == b && std::stoull(header_value(h, "end")) == e,
            path, ": chunk range does not match the plan");
    require(std::stoi(header_value(h, "frames")) == n_frames, path, ": frame count mismatch");
    const int na = std::stoi(header_value(h, "n_angles"));
    std::vector<std::complex<double>> data = as_complex_f64(payload);
    const std::size_t len = e - b;
    require(data.size() == len * static_cast<std::size_t>(n_frames), path,
            ": payload does not match the chunk shape");
    for (int f = 0; f < n_frames; ++f) {
      out[f].n_angles = na;
      std::copy(data.begin() + f * len, data.begin() + (f + 1) * len, out[f].values.begin() + b);
    }
  }
  return out;
}

void write_iq_volume(const std::string& path, const IqVolume& vol) {
  require(vol.values.size() == vol.grid.num_points(), "volume values do not match the grid dims");
  const GridSpec& g = vol.grid;
  ContainerHeader h{
      {"kind", "iq_volume"},
      {"dims", detail::concat(g.dims[0], ' ', g.dims[1], ' ', g.dims[2])},
      {"spacing", fmt17(g.spacing.x) + " " + fmt17(g.spacing.y) + " " + fmt17(g.spacing.z)},
      {"origin", fmt17(g.origin.x) + " " + fmt17(g.origin.y) + " " + fmt17(g.origin.z)},
      {"frame", std::to_string(vol.frame_index + 1)},
      {"n_angles", std::to_string(vol.n_angles)}};
  write_container(path, h, make_payload(std::span<const std::complex<double>>(vol.values)));
}

IqVolume read_iq_volume(const std::string& path) {
  auto [h, payload] = read_container(path);
  require(header_value(h, "kind") == "iq_volume", path, ": not a volume container");
  IqVolume v;
  std::istringstream is(header_value(h, "dims"));
  is >> v.grid.dims[0] >> v.grid.dims[1] >> v.grid.dims[2];
  require(!is.fail(), path, ": bad dims header");
  double sp[3], org[3];
  parse3(header_value(h, "spacing"), sp);
  parse3(header_value(h, "origin"), org);
  v.grid.spacing = {sp[0], sp[1], sp[2]};
  v.grid.origin = {org[0], org[1], org[2]};
  v.frame_index = std::stoi(header_value(h, "frame")) - 1;
  v.n_angles = std::stoi(header_value(h, "n_angles"));
  v.values = as_complex_f64(payload);
  require(v.values.size() == v.grid.num_points(), path, ": payload does not match the grid dims");
  return v;
}

}  // namespace beamform

namespace post {

namespace {
void check_frames(const std::vector<beamform::IqVolume>& ens, const char* who) {
  const auto& first = ens.front();
  std::size_t n = first.grid.num_points();
  require(n > 0, who, " needs a nonempty grid");
  for (const auto& fr : ens) {
    require(fr.grid.dims == first.grid.dims, "ensemble frames must share one grid");
    require(fr.values.size() == n, "frame value count must match the grid");
  }
}

std::vector<std::complex<float>> casorati(const std::vector<beamform::IqVolume>& ens) {
  std::size_t n = ens.front().grid.num_points();
  std::vector<std::complex<float>> x(ens.size() * n);
  for (std::size_t f = 0; f < ens.size(); ++f)
    std::copy(ens[f].values.begin(), ens[f].values.end(), x.begin() + f * n);
  return x;
}
}  // namespace

// svd.cpp:29-93.
std::vector<beamform::IqVolume> svd_filter(const std::vector<beamform::IqVolume>& ensemble,
                                           int keep_lo, int keep_hi, SvdReport* report) {
  require(!ensemble.empty(), "svd_filter needs a nonempty ensemble");
  check_frames(ensemble, "svd_filter");
  require(ensemble.size() >= 2, "svd_filter needs at least two frames");
  const std::size_t n = ensemble.front().grid.num_points();
  require(ensemble.size() <= n, "svd_filter needs at least as many voxels as frames");
  const int F = static_cast<int>(ensemble.size());
  require(keep_lo >= 1 && keep_lo <= keep_hi && keep_hi <= F,
          "retained band must satisfy 1 <= lo <= hi <= frames, got [", keep_lo, ", ", keep_hi,
          "] with ", F, " frames");
  std::vector<std::complex<float>> x = casorati(ensemble), y(x.size());
  std::vector<double> sigma(F), corr(report ? static_cast<std::size_t>(F) * F : 0);
  ok(fqfg_svd_filter(reinterpret_cast<const float*>(x.data()), F, n, keep_lo, keep_hi,
                     reinterpret_cast<float*>(y.data()), sigma.data(), nullptr,
                     report ? corr.data() : nullptr));
  if (report) {
    report->n_modes = F;
    report->keep_lo = keep_lo;
    report->keep_hi = keep_hi;
    report->singular_values = sigma;
    report->mode_correlation = corr;
  }
  std::vector<beamform::IqVolume> out(F);
  for (int f = 0; f < F; ++f) {
    out[f].grid = ensemble[f].grid;
    out[f].frame_index = ensemble[f].frame_index;
    out[f].n_angles = ensemble[f].n_angles;
    out[f].values.assign(y.begin() + static_cast<std::size_t>(f) * n,
                         y.begin() + static_cast<std::size_t>(f + 1) * n);
  }
  return out;
}

// render.cpp:23-42.
VoxelGrid power_doppler(const std::vector<beamform::IqVolume>& ensemble) {
  require(!ensemble.empty(), "power_doppler needs at least one frame");
  check_frames(ensemble, "power_doppler");
  const auto& g = ensemble.front().grid;
  std::vector<std::complex<float>> x = casorati(ensemble);
  VoxelGrid pd(g.dims, g.spacing, g.origin);
  ok(fqfg_power_doppler(reinterpret_cast<const float*>(x.data()),
                        static_cast<int>(ensemble.size()), g.num_points(), pd.data().data()));
  return pd;
}

// render.cpp:44-68.
VoxelGrid render_db(const VoxelGrid& volume, double dynamic_range_db, DbScale scale) {
  require(volume.components() == 1, "render_db expects a scalar volume");
  require(!volume.data().empty(), "render_db needs a nonempty volume");
  VoxelGrid out(volume.dims(), volume.spacing(), volume.origin());
  ok(fqfg_render_db(volume.data().data(), volume.dims().data(), dynamic_range_db,
                    scale == DbScale::power ? 1 : 0, out.data().data()));
  return out;
}

// render.cpp:70-78.
VoxelGrid bmode(const beamform::IqVolume& iq, double dynamic_range_db) {
  std::size_t n = iq.grid.num_points();
  require(n > 0 && iq.values.size() == n, "bmode needs an IQ volume matching its grid");
  VoxelGrid out(iq.grid.dims, iq.grid.spacing, iq.grid.origin);
  ok(fqfg_bmode(reinterpret_cast<const double*>(iq.values.data()), iq.grid.dims.data(),
                dynamic_range_db, out.data().data()));
  return out;
}

// render.cpp:80-104.
VoxelGrid mip(const VoxelGrid& volume, int axis) {
  require(axis >= 0 && axis < 3, "mip axis must be 0, 1, or 2, got ", axis);
  require(volume.components() == 1, "mip expects a scalar volume");
  require(!volume.data().empty(), "mip needs a nonempty volume");
  auto out_dims = volume.dims();
  out_dims[axis] = 1;
  VoxelGrid out(out_dims, volume.spacing(), volume.origin());
  ok(fqfg_mip(volume.data().data(), volume.dims().data(), axis, out.data().data()));
  return out;
}

// render.cpp:106-145.
VoxelGrid ground_truth_pd(const std::vector<std::vector<Vec3>>& positions_per_frame,
                          const beamform::GridSpec& grid, double sigma_voxels) {
  require(!positions_per_frame.empty(), "ground_truth_pd needs at least one frame");
  require(grid.num_points() > 0, "ground_truth_pd needs a nonempty grid");
  require(sigma_voxels > 0.0, "kernel sigma must be positive, got ", sigma_voxels);
  std::vector<double> xyz;
  std::vector<int> counts;
  for (const auto& frame : positions_per_frame) {
    counts.push_back(static_cast<int>(frame.size()));
    for (const auto& p : frame) xyz.insert(xyz.end(), {p.x, p.y, p.z});
  }
  fqfg_grid g{{grid.dims[0], grid.dims[1], grid.dims[2]},
              {grid.spacing.x, grid.spacing.y, grid.spacing.z},
              {grid.origin.x, grid.origin.y, grid.origin.z}};
  VoxelGrid out(grid.dims, grid.spacing, grid.origin);
  ok(fqfg_ground_truth_pd(xyz.data(), counts.data(), static_cast<int>(counts.size()), &g,
                          sigma_voxels, out.data().data()));
  return out;
}

// metrics.cpp:84-101.
MetricsReport metrics(const VoxelGrid& test, const VoxelGrid& reference) {
  require(test.components() == 1 && reference.components() == 1,
          "metrics expects scalar images");
  require(test.dims() == reference.dims(), "metrics needs images of identical shape");
  require(!test.data().empty(), "metrics needs nonempty images");
  double r[3];
  ok(fqfg_metrics(test.data().data(), reference.data().data(), test.dims().data(), r));
  MetricsReport m;
  m.mse = r[0];
  m.psnr = r[1];
  m.ssim = r[2];
  return m;
}

}  // namespace post
}  // namespace fqf
