// test_dropin.cpp -- the reference's own beamform/post test cases
// (proj/tests/test_beamform.cpp, test_post.cpp) restated against the GPU
// drop-in (fqf_dropin.cpp + libfqfgpu.so).  Same fixtures, same seeded
// libstdc++ engines, same API calls; tolerances relaxed only where the
// reference compares FP64 against FP64 and the GPU computes in f32 (each
// such place says so).  Run by tests/test_dropin_cpp.py on a B200.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "fqf/beamform/das.hpp"
#include "fqf/beamform/iq.hpp"
#include "fqf/core/error.hpp"
#include "fqf/post/metrics.hpp"
#include "fqf/post/render.hpp"
#include "fqf/post/svd.hpp"
#include "fqf/rf/simulate.hpp"
#include "fqf/rf/transducer.hpp"
#include "fqf/tissue/cloud.hpp"

using namespace fqf;
using namespace fqf::beamform;
using rf::RfFrame;
using rf::Transducer;
using rf::TxEvent;
using cd = std::complex<double>;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(c)) {                                                           \
      ++g_fail;                                                           \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
    }                                                                     \
  } while (0)
#define CHECK_THROWS(expr)                                   \
  do {                                                       \
    bool thrown_ = false;                                    \
    try {                                                    \
      (void)(expr);                                          \
    } catch (const Error&) {                                 \
      thrown_ = true;                                        \
    }                                                        \
    CHECK(thrown_);                                          \
  } while (0)

static void run(const char* name, const std::function<void()>& fn) {
  int before = g_fail;
  try {
    fn();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("  FAIL exception: %s\n", e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

constexpr double kPi = 3.14159265358979323846;
// f32 IQ and accumulation vs the reference's FP64.
constexpr double kIqTol = 1e-5;

static Transducer small_probe(int n, double fc) {
  Transducer t;
  t.name = "test";
  t.pitch = 0.3e-3;
  t.half_width = 0.135e-3;
  t.subelements = 2;
  t.center_frequency = fc;
  t.fractional_bandwidth = 0.6;
  for (int i = 0; i < n; ++i) t.elements.push_back({(i - (n - 1) / 2.0) * t.pitch, 0.0, 0.0});
  return t;
}

static RfFrame make_frame(int T, int E, double fs, double t0, const TxEvent& tx) {
  RfFrame f;
  f.n_samples = T;
  f.n_elements = E;
  f.sampling_rate = fs;
  f.t0 = t0;
  f.tx = tx;
  f.samples.assign(static_cast<std::size_t>(T) * E, 0.0);
  return f;
}

static TxEvent zero_tx(int n, double angle = 0.0) {
  TxEvent tx;
  tx.angle = angle;
  tx.delays.assign(n, 0.0);
  tx.apodization.assign(n, 1.0);
  return tx;
}

static double max_rel_diff(const std::vector<cd>& a, const std::vector<cd>& b) {
  double s = 0, m = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s = std::max({s, std::abs(a[i]), std::abs(b[i])});
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return s == 0 ? 0 : m / s;
}

// test_beamform.cpp:68-118 restated: literal per-voxel DAS over rf_to_iq.
static std::vector<cd> literal_das(const std::vector<std::vector<RfFrame>>& frames, int frame,
                                   const GridSpec& grid, const Transducer& td,
                                   const BeamformParams& bp) {
  std::vector<cd> out(grid.num_points(), {0, 0});
  int na = static_cast<int>(frames[frame].size());
  for (int a = 0; a < na; ++a) {
    const RfFrame& r = frames[frame][a];
    IqFrame iq = rf_to_iq(r, bp.center_frequency, bp.lowpass_taps);
    double sa = std::sin(r.tx.angle), ca = std::cos(r.tx.angle);
    double ref = std::numeric_limits<double>::infinity();
    for (const Vec3& el : td.elements) ref = std::min(ref, el.x * sa);
    for (std::size_t v = 0; v < out.size(); ++v) {
      Vec3 p = grid.point(v);
      double ttx = (p.x * sa + p.z * ca - ref) / bp.c;
      cd acc{0, 0};
      for (int e = 0; e < td.n_elements(); ++e) {
        const Vec3& el = td.elements[e];
        if (bp.f_number > 0.0 && std::hypot(p.x - el.x, p.y - el.y) * 2.0 * bp.f_number > p.z - el.z)
          continue;
        double tau = ttx + norm(p - el) / bp.c;
        double s = (tau - r.t0) * r.sampling_rate;
        double sfl = std::floor(s), frac = s - sfl;
        int i0 = static_cast<int>(sfl);
        cd val{0, 0};
        if (i0 >= 0 && i0 < r.n_samples) val += (1.0 - frac) * iq.at(i0, e);
        if (frac > 0.0 && i0 + 1 >= 0 && i0 + 1 < r.n_samples) val += frac * iq.at(i0 + 1, e);
        acc += val * std::polar(1.0, 2.0 * kPi * bp.center_frequency * tau);
      }
      out[v] += acc;
    }
  }
  for (auto& v : out) v /= static_cast<double>(na);
  return out;
}

int main() {
  run("chunk plan follows the accumulator byte formula", [] {
    CHECK(plan_chunks(1'000'000, 5, 100'000'000).n_chunks == 1);
    ChunkPlan q = plan_chunks(1'000'000, 5, 10'000'000);
    CHECK(q.n_chunks == 8 && q.ranges.back().second == 1'000'000);
    CHECK(plan_chunks(3, 1, 24).n_chunks == 3);
    CHECK_THROWS(plan_chunks(0, 5, 1'000));
    CHECK_THROWS(plan_chunks(100, 5, 80));
  });

  run("demodulation maps an in-band tone to a constant baseband value", [] {
    double fc = 5e6, fs = 20e6;
    RfFrame f = make_frame(400, 2, fs, 0.0, zero_tx(2));
    for (int t = 0; t < 400; ++t) {
      f.at(t, 0) = std::cos(2 * kPi * fc * t / fs);
      f.at(t, 1) = std::cos(2 * kPi * fc * t / fs + kPi / 3);
    }
    IqFrame iq = rf_to_iq(f, fc);
    CHECK(iq.n_samples == 400 && iq.n_elements == 2 && iq.center_frequency == fc);
    for (int t = 40; t < 360; ++t) {
      CHECK(std::abs(iq.at(t, 0) - 1.0) < 0.01);
      CHECK(std::abs(iq.at(t, 1) - std::polar(1.0, kPi / 3)) < 0.01);
    }
  });

  run("demodulation is linear and exact for power-of-two scaling", [] {
    std::mt19937 rng(17);
    std::uniform_real_distribution<double> d(-1, 1);
    RfFrame base = make_frame(128, 3, 20e6, 0.0, zero_tx(3));
    for (auto& s : base.samples) s = d(rng);
    RfFrame twice = base;
    for (auto& s : twice.samples) s *= 2.0;
    IqFrame a = rf_to_iq(base, 5e6), b = rf_to_iq(twice, 5e6);
    // Bitwise: the x2 input scaling is exact in f32 as in FP64.
    for (std::size_t i = 0; i < a.samples.size(); ++i) CHECK(b.samples[i] == 2.0 * a.samples[i]);
    CHECK_THROWS(rf_to_iq(make_frame(64, 1, 19e6, 0, zero_tx(1)), 9.5e6));
    CHECK_THROWS(rf_to_iq(make_frame(64, 1, 20e6, 0, zero_tx(1)), 5e6, 32));
  });

  run("delay matrix places on-axis echoes at the round-trip sample", [] {
    double c = 1024.0, fs = 2097152.0, fc = 262144.0;
    Transducer td = small_probe(1, fc);
    td.elements = {{0, 0, 0}};
    BeamformParams bp;
    bp.c = c;
    bp.center_frequency = fc;
    bp.f_number = 0.0;
    double z = 40.0 * c / (2.0 * fs);
    std::vector<Vec3> vox = {{0, 0, z}};
    DelayMatrix m = build_delay_matrix(vox, zero_tx(1), td, bp, fs, 0.0, 128);
    CHECK(m.row_ptr == std::vector<std::size_t>({0, 1}) && m.col_idx[0] == 40);
    CHECK(std::abs(m.values[0] - std::polar(1.0, 2 * kPi * fc * (2 * z / c))) < 1e-12);
    CHECK(m.out_of_window == 0 && m.padded_samples == 128);
    vox = {{0, 0, 40.5 * c / (2.0 * fs)}};
    m = build_delay_matrix(vox, zero_tx(1), td, bp, fs, 0.0, 128);
    CHECK(m.row_ptr[1] == 2 && m.col_idx[0] == 40 && m.col_idx[1] == 41);
    CHECK(std::abs(std::abs(m.values[0]) - 0.5) < 1e-15);
    bp.interp_order = 0;
    vox = {{0, 0, 40.25 * c / (2.0 * fs)}};
    m = build_delay_matrix(vox, zero_tx(1), td, bp, fs, 0.0, 128);
    CHECK(m.row_ptr[1] == 1 && m.col_idx[0] == 40);
    bp.interp_order = 1;
    vox = {{0, 0, 200.0 * c / (2.0 * fs)}};
    m = build_delay_matrix(vox, zero_tx(1), td, bp, fs, 0.0, 128);
    CHECK(m.row_ptr[1] == 0 && m.out_of_window == 1 && m.padded_samples > m.recorded_samples);
    vox = {{0, 0, 40.0 * c / (2.0 * fs)}};
    m = build_delay_matrix(vox, zero_tx(1), td, bp, fs, 64.0 / fs, 128);
    CHECK(m.row_ptr[1] == 0 && m.out_of_window == 1);
  });

  run("delay matrix honors the receive f-number aperture", [] {
    Transducer td = small_probe(1, 5e6);
    td.elements = {{0, 0, 0}, {0.9e-3, 0, 0}, {-0.9e-3, 0, 0}, {1.1e-3, 0, 0}, {-1.1e-3, 0, 0}};
    BeamformParams bp;
    bp.center_frequency = 5e6;
    std::vector<Vec3> vox = {{0, 0, 3.0e-3}};
    DelayMatrix m = build_delay_matrix(vox, zero_tx(5), td, bp, 20e6, 0.0, 512);
    std::vector<bool> seen(5, false);
    for (std::size_t i = m.row_ptr[0]; i < m.row_ptr[1]; ++i) seen[m.col_idx[i] % 5] = true;
    CHECK(seen == std::vector<bool>({true, true, true, false, false}));
  });

  run("apply_delay_matrix equals the per-entry sum", [] {
    Transducer td = small_probe(16, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    bp.f_number = 1.2;
    std::mt19937 rng(23);
    std::uniform_real_distribution<double> ux(-3e-3, 3e-3), uz(2e-3, 14e-3), d(-1, 1);
    std::vector<Vec3> vox;
    for (int i = 0; i < 60; ++i) vox.push_back({ux(rng), 0.0, uz(rng)});
    TxEvent tx = rf::plane_wave_delays(td, 4.0 * kPi / 180.0, 1540.0);
    DelayMatrix m = build_delay_matrix(vox, tx, td, bp, 20e6, 0.0, 512);
    IqFrame iq;
    iq.n_samples = 512;
    iq.n_elements = 16;
    for (int i = 0; i < 512 * 16; ++i) iq.samples.push_back({d(rng), d(rng)});
    std::vector<cd> y(m.rows);
    apply_delay_matrix(m, iq, y.data());
    for (std::size_t r = 0; r < m.rows; ++r) {
      cd acc{0, 0};
      for (std::size_t i = m.row_ptr[r]; i < m.row_ptr[r + 1]; ++i)
        acc += m.values[i] * iq.samples[m.col_idx[i]];
      CHECK(y[r] == acc);  // same FP64 operations in entry order
      for (std::size_t i = m.row_ptr[r]; i < m.row_ptr[r + 1]; ++i)
        CHECK(std::abs(m.values[i]) <= 1.0 + 1e-12);
    }
  });

  run("reconstruction matches the literal per-voxel reference", [] {
    double fc = 5e6, fs = 20e6;
    Transducer td = small_probe(8, fc);
    BeamformParams bp;
    bp.center_frequency = fc;
    std::mt19937 rng(31);
    std::uniform_real_distribution<double> d(-1, 1);
    std::vector<std::vector<RfFrame>> frames(2);
    for (int f = 0; f < 2; ++f)
      for (double a : {-3.0 * kPi / 180.0, 2.0 * kPi / 180.0}) {
        RfFrame fr = make_frame(64, 8, fs, 0.25e-6, rf::plane_wave_delays(td, a, bp.c));
        for (auto& s : fr.samples) s = d(rng);
        frames[f].push_back(fr);
      }
    GridSpec grid;
    grid.dims = {7, 2, 5};
    grid.spacing = {0.2e-3, 0.3e-3, 0.2e-3};
    grid.origin = {-0.6e-3, -0.15e-3, 1.2e-3};
    DasOptions opts;
    opts.memory_budget_bytes = 16ull * 24 * 2;
    DasStats st;
    auto vols = das_reconstruct(frames, grid, td, bp, opts, &st);
    CHECK(vols.size() == 2 && st.chunks == 3 && st.matrix_builds == 6);
    CHECK(st.accumulator_bytes_peak <= opts.memory_budget_bytes);
    for (int f = 0; f < 2; ++f) {
      CHECK(vols[f].frame_index == f && vols[f].n_angles == 2);
      CHECK(max_rel_diff(vols[f].values, literal_das(frames, f, grid, td, bp)) < kIqTol);
    }
    // SURVEY.md 8(c) golden values from the reference build.
    CHECK(std::abs(vols[0].values[0] - cd(0.21767054125126079, -0.23091352539589127)) < 1e-5);
    CHECK(std::abs(vols[1].values[0] - cd(-0.2515352884279673, 0.01450684879472558)) < 1e-5);
  });

  run("any chunk partition reconstructs the same volume; caching changes nothing", [] {
    Transducer td = small_probe(8, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    std::mt19937 rng(41);
    std::uniform_real_distribution<double> d(-1, 1);
    std::vector<std::vector<RfFrame>> frames(1);
    for (double a : {-2.0 * kPi / 180.0, 3.0 * kPi / 180.0}) {
      RfFrame fr = make_frame(96, 8, 20e6, 0.0, rf::plane_wave_delays(td, a, bp.c));
      for (auto& s : fr.samples) s = d(rng);
      frames[0].push_back(fr);
    }
    GridSpec grid;
    grid.dims = {21, 1, 11};
    grid.spacing = {0.15e-3, 0.2e-3, 0.25e-3};
    grid.origin = {-1.5e-3, 0.0, 1.5e-3};
    std::vector<cd> base;
    for (int target : {1, 3, 7}) {
      DasOptions opts;
      opts.memory_budget_bytes = (16ull * grid.num_points() * 2 + target - 1) / target;
      DasStats st;
      auto v = das_reconstruct(frames, grid, td, bp, opts, &st);
      CHECK(st.chunks == target);
      if (target == 1)
        base = v[0].values;
      else
        CHECK(v[0].values == base);  // bitwise on the GPU (reference bound 1e-7)
      opts.cache_matrices = false;
      CHECK(das_reconstruct(frames, grid, td, bp, opts)[0].values == base);
    }
  });

  run("averaging identical transmits reproduces the single-transmit volume", [] {
    Transducer td = small_probe(6, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    std::mt19937 rng(47);
    std::uniform_real_distribution<double> d(-1, 1);
    RfFrame fr = make_frame(80, 6, 20e6, 0.0, rf::plane_wave_delays(td, 0.0, bp.c));
    for (auto& s : fr.samples) s = d(rng);
    GridSpec grid;
    grid.dims = {9, 1, 7};
    grid.spacing = {0.2e-3, 0.2e-3, 0.2e-3};
    grid.origin = {-0.8e-3, 0.0, 1.0e-3};
    auto v1 = das_reconstruct({{fr}}, grid, td, bp);
    auto v2 = das_reconstruct({{fr, fr}}, grid, td, bp);
    // Exact in FP64 (mean of equal terms); f32 sums both angles per element.
    CHECK(max_rel_diff(v1[0].values, v2[0].values) < 1e-6);
    CHECK(v2[0].n_angles == 2);
  });

  run("reconstruction is linear in the radio-frequency input", [] {
    Transducer td = small_probe(6, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    std::mt19937 rng(53);
    std::uniform_real_distribution<double> d(-1, 1);
    TxEvent tx = rf::plane_wave_delays(td, 1.5 * kPi / 180.0, bp.c);
    RfFrame f1 = make_frame(72, 6, 20e6, 0.0, tx), f2 = make_frame(72, 6, 20e6, 0.0, tx);
    for (auto& s : f1.samples) s = d(rng);
    for (auto& s : f2.samples) s = d(rng);
    RfFrame mix = f1;
    for (std::size_t i = 0; i < mix.samples.size(); ++i)
      mix.samples[i] = 2.0 * f1.samples[i] + f2.samples[i];
    GridSpec grid;
    grid.dims = {11, 1, 9};
    grid.spacing = {0.15e-3, 0.2e-3, 0.2e-3};
    grid.origin = {-0.75e-3, 0.0, 0.8e-3};
    auto a = das_reconstruct({{f1}}, grid, td, bp), b = das_reconstruct({{f2}}, grid, td, bp),
         m = das_reconstruct({{mix}}, grid, td, bp);
    std::vector<cd> expect(a[0].values.size());
    for (std::size_t i = 0; i < expect.size(); ++i) expect[i] = 2.0 * a[0].values[i] + b[0].values[i];
    CHECK(max_rel_diff(m[0].values, expect) < 1e-6);  // reference bound 1e-9 in FP64
  });

  run("volume files round-trip and chunk files drive assembly", [] {
    Transducer td = small_probe(4, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    std::mt19937 rng(61);
    std::uniform_real_distribution<double> d(-1, 1);
    std::vector<std::vector<RfFrame>> frames(2);
    for (int f = 0; f < 2; ++f) {
      RfFrame fr = make_frame(48, 4, 20e6, 0.0, rf::plane_wave_delays(td, 0.0, bp.c));
      for (auto& s : fr.samples) s = d(rng);
      frames[f].push_back(fr);
    }
    GridSpec grid;
    grid.dims = {6, 1, 5};
    grid.spacing = {0.2e-3, 0.2e-3, 0.2e-3};
    grid.origin = {-0.5e-3, 0.0, 1.0e-3};
    std::size_t n = grid.num_points();
    auto dir = (std::filesystem::temp_directory_path() / "fqf_dropin_tests" / "assembly").string();
    std::filesystem::remove_all(dir);
    DasOptions opts;
    opts.memory_budget_bytes = 16ull * ((n + 1) / 2);
    opts.work_dir = dir;
    opts.write_frames = true;
    opts.keep_chunk_files = true;
    auto vols = das_reconstruct(frames, grid, td, bp, opts);
    for (int f = 0; f < 2; ++f) {
      IqVolume rd = read_iq_volume(dir + "/Frame_" + std::to_string(f + 1) + ".fqf");
      CHECK(rd.frame_index == f && rd.n_angles == 1 && rd.grid.dims == grid.dims);
      CHECK(rd.values == vols[f].values);
    }
    ChunkPlan plan = plan_chunks(n, 1, opts.memory_budget_bytes);
    auto again = assemble_frames(dir, plan, grid, 2);
    for (int f = 0; f < 2; ++f) CHECK(again[f].values == vols[f].values);
    std::filesystem::remove(dir + "/IQ_CHUNK_2.fqf");
    bool named = false;
    try {
      assemble_frames(dir, plan, grid, 2);
    } catch (const Error& e) {
      named = std::string(e.what()).find("IQ_CHUNK_2") != std::string::npos;
    }
    CHECK(named);
  });

  run("reconstruction rejects inconsistent inputs; out-of-window stays finite", [] {
    Transducer td = small_probe(4, 5e6);
    BeamformParams bp;
    bp.center_frequency = 5e6;
    GridSpec grid;
    grid.dims = {4, 1, 4};
    grid.spacing = {0.2e-3, 0.2e-3, 0.2e-3};
    grid.origin = {-0.3e-3, 0.0, 1.0e-3};
    TxEvent tx = rf::plane_wave_delays(td, 0.0, bp.c);
    RfFrame good = make_frame(32, 4, 20e6, 0.0, tx);
    CHECK_THROWS(das_reconstruct({}, grid, td, bp));
    CHECK_THROWS(das_reconstruct({{good}, {make_frame(32, 4, 18e6, 0.0, tx)}}, grid, td, bp));
    CHECK_THROWS(das_reconstruct({{good, good}, {good}}, grid, td, bp));
    CHECK_THROWS(das_reconstruct({{make_frame(32, 3, 20e6, 0.0, tx)}}, grid, td, bp));
    DasOptions small;
    small.memory_budget_bytes = 16;
    CHECK_THROWS(das_reconstruct({{good}}, grid, td, bp, small));
    RfFrame fr = make_frame(24, 4, 20e6, 0.0, tx);
    std::mt19937 rng(71);
    std::uniform_real_distribution<double> d(-1, 1);
    for (auto& s : fr.samples) s = d(rng);
    GridSpec deep;
    deep.dims = {3, 1, 4};
    deep.spacing = {0.2e-3, 0.2e-3, 2.0e-3};
    deep.origin = {-0.2e-3, 0.0, 1.0e-3};
    DasStats st;
    auto v = das_reconstruct({{fr}}, deep, td, bp, {}, &st);
    CHECK(st.out_of_window > 0);
    for (const auto& x : v[0].values) CHECK(std::isfinite(x.real()) && std::isfinite(x.imag()));
  });

  auto ensemble = [](const GridSpec& g, int frames, const std::function<cd(int, std::size_t)>& fill) {
    std::vector<IqVolume> out(frames);
    for (int f = 0; f < frames; ++f) {
      out[f].grid = g;
      out[f].frame_index = f;
      out[f].n_angles = 1;
      for (std::size_t v = 0; v < g.num_points(); ++v) out[f].values.push_back(fill(f, v));
    }
    return out;
  };
  auto grid3 = [](int nx, int ny, int nz) {
    GridSpec g;
    g.dims = {nx, ny, nz};
    g.spacing = {1e-4, 1e-4, 1e-4};
    return g;
  };
  auto fro = [](const std::vector<IqVolume>& e) {
    double s = 0;
    for (const auto& v : e)
      for (const auto& z : v.values) s += std::norm(z);
    return std::sqrt(s);
  };

  run("svd filter removes a static ensemble and keeps identity", [&] {
    auto g = grid3(10, 1, 20);
    std::mt19937_64 rng(401);
    std::normal_distribution<double> nd;
    std::vector<cd> pattern(g.num_points());
    for (auto& z : pattern) z = {nd(rng), nd(rng)};
    auto ens = ensemble(g, 6, [&](int, std::size_t v) { return pattern[v]; });
    double scale = fro(ens);
    post::SvdReport rep;
    auto high = post::svd_filter(ens, 2, 6, &rep);
    // f32 ensemble: residual ~1e-7 of the input (reference: 1e-9 in FP64).
    CHECK(fro(high) <= 1e-6 * scale);
    CHECK(std::abs(rep.singular_values[0] - scale) <= 1e-6 * scale);
    CHECK(rep.keep_lo == 2 && rep.keep_hi == 6 && rep.n_modes == 6);
    auto all = post::svd_filter(ens, 1, 6);
    double diff = 0;
    for (int f = 0; f < 6; ++f)
      for (std::size_t v = 0; v < g.num_points(); ++v) diff += std::norm(all[f].values[v] - ens[f].values[v]);
    CHECK(std::sqrt(diff) <= 1e-6 * scale);
  });

  run("svd bands conserve energy; correlation symmetric with unit diagonal", [&] {
    auto g = grid3(15, 2, 10);
    std::mt19937_64 rng(402);
    std::normal_distribution<double> nd;
    auto ens = ensemble(g, 7, [&](int, std::size_t) { return cd{nd(rng), nd(rng)}; });
    post::SvdReport rep;
    auto low = post::svd_filter(ens, 1, 3, &rep);
    auto high = post::svd_filter(ens, 4, 7);
    double energy = fro(ens) * fro(ens), spectral = 0;
    for (double s : rep.singular_values) spectral += s * s;
    CHECK(std::abs(spectral - energy) <= 1e-6 * energy);
    for (std::size_t j = 0; j + 1 < rep.singular_values.size(); ++j)
      CHECK(rep.singular_values[j] >= rep.singular_values[j + 1] && rep.singular_values[j + 1] >= 0);
    double diff = 0;
    for (int f = 0; f < 7; ++f)
      for (std::size_t v = 0; v < g.num_points(); ++v)
        diff += std::norm(low[f].values[v] + high[f].values[v] - ens[f].values[v]);
    CHECK(std::sqrt(diff) <= 1e-6 * fro(ens));
    const auto& c = rep.mode_correlation;
    CHECK(c.size() == 49);
    for (int i = 0; i < 7; ++i) {
      CHECK(std::abs(c[i * 7 + i] - 1.0) < 1e-12);
      for (int j = 0; j < 7; ++j) CHECK(std::abs(c[i * 7 + j] - c[j * 7 + i]) <= 1e-12 && std::abs(c[i * 7 + j]) <= 1 + 1e-12);
    }
  });

  run("svd filter raises the in-vessel power fraction", [&] {
    auto g = grid3(20, 1, 20);
    std::mt19937_64 rng(404);
    std::normal_distribution<double> nd;
    std::vector<cd> tissue(g.num_points());
    for (auto& z : tissue) z = cd{nd(rng), nd(rng)} * 100.0;
    auto in_vessel = [](std::size_t v) { return v % 20 == 8 || v % 20 == 9; };
    auto ens = ensemble(g, 10, [&](int, std::size_t v) {
      cd z = tissue[v];
      if (in_vessel(v)) z += cd{nd(rng), nd(rng)};
      return z;
    });
    auto frac = [&](const VoxelGrid& pd) {
      double m = 0, t = 0;
      for (std::size_t v = 0; v < g.num_points(); ++v) {
        t += pd.data()[v];
        if (in_vessel(v)) m += pd.data()[v];
      }
      return m / t;
    };
    double before = frac(post::power_doppler(ens));
    double after = frac(post::power_doppler(post::svd_filter(ens, 2, 10)));
    CHECK(before < 0.3 && after > 0.9 && after > before);
  });

  run("svd filter rejects degenerate input; power doppler sums |IQ|^2", [&] {
    auto g = grid3(4, 1, 4);
    auto ens = ensemble(g, 3, [](int f, std::size_t v) { return cd(f + 1.0, double(v)); });
    CHECK_THROWS(post::svd_filter({}, 1, 1));
    CHECK_THROWS(post::svd_filter(std::vector<IqVolume>(ens.begin(), ens.begin() + 1), 1, 1));
    CHECK_THROWS(post::svd_filter(ens, 0, 2));
    CHECK_THROWS(post::svd_filter(ens, 1, 4));
    CHECK_THROWS(post::svd_filter(ens, 3, 2));
    CHECK_THROWS(post::svd_filter(ensemble(g, 3, [](int, std::size_t) { return cd{}; }), 1, 3));
    CHECK_THROWS(post::svd_filter(ensemble(grid3(1, 1, 2), 3, [](int f, std::size_t v) { return cd(f + 1.0, v + 1.0); }), 1, 3));
    auto g2 = grid3(6, 1, 5);
    const cd lattice[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    auto unit = ensemble(g2, 100, [&](int f, std::size_t v) { return lattice[(f + v) % 4]; });
    VoxelGrid pd = post::power_doppler(unit);
    CHECK(pd.dims() == (std::array<int, 3>{6, 1, 5}));
    for (double v : pd.data()) CHECK(v == 100.0);
    CHECK_THROWS(post::power_doppler({}));
  });

  // ---- display and scoring (test_post.cpp:318-501), now on the GPU ----
  run("render_db maps peak to one and the floor to zero", [&] {
    VoxelGrid v({4, 1, 1}, {1, 1, 1}, {0, 0, 0});
    v.data() = {2.0, 1.0, 2e-9, 0.0};
    VoxelGrid amp = post::render_db(v, 60.0, post::DbScale::amplitude);
    CHECK(amp.at(0, 0, 0) == 1.0);
    CHECK(std::abs(amp.at(1, 0, 0) - (60.0 - 20.0 * std::log10(2.0)) / 60.0) <= 1e-14);
    CHECK(amp.at(2, 0, 0) == 0.0 && amp.at(3, 0, 0) == 0.0);
    VoxelGrid pw = post::render_db(v, 60.0, post::DbScale::power);
    CHECK(pw.at(0, 0, 0) == 1.0);
    CHECK(std::abs(pw.at(1, 0, 0) - (60.0 - 10.0 * std::log10(2.0)) / 60.0) <= 1e-14);
    VoxelGrid zeros({3, 1, 1}, {1, 1, 1}, {0, 0, 0});
    CHECK_THROWS(post::render_db(zeros, 60.0, post::DbScale::amplitude));
    CHECK_THROWS(post::render_db(v, 0.0, post::DbScale::amplitude));
    CHECK_THROWS(post::render_db(v, -5.0, post::DbScale::amplitude));
  });

  run("render_db preserves intensity ordering; bmode renders the envelope", [&] {
    VoxelGrid v({50, 1, 1}, {1, 1, 1}, {0, 0, 0});
    std::mt19937 rng(5);
    std::uniform_real_distribution<double> u(0.0, 10.0);
    for (double& x : v.data()) x = u(rng);
    VoxelGrid r = post::render_db(v, 40.0, post::DbScale::power);
    for (int i = 0; i < 50; ++i)
      for (int j = 0; j < 50; ++j)
        if (v.data()[i] < v.data()[j]) CHECK(r.data()[i] <= r.data()[j]);
    auto g = grid3(3, 2, 2);
    auto flat = ensemble(g, 1, [](int, std::size_t v) { return std::polar(2.0, 0.3 * v); });
    VoxelGrid img = post::bmode(flat.front(), 75.0);
    for (double x : img.data()) CHECK(std::abs(x - 1.0) <= 1e-12);
    IqVolume bad = flat.front();
    bad.values.pop_back();
    CHECK_THROWS(post::bmode(bad, 75.0));
  });

  run("mip collapses one axis to its maximum", [&] {
    VoxelGrid v({4, 3, 2}, {1, 2, 3}, {0.5, 0.25, 0.125});
    std::mt19937 rng(9);
    std::normal_distribution<double> nd;
    for (double& x : v.data()) x = nd(rng);
    for (int axis = 0; axis < 3; ++axis) {
      VoxelGrid m = post::mip(v, axis);
      auto want = v.dims();
      want[axis] = 1;
      CHECK(m.dims() == want && m.spacing().x == v.spacing().x && m.origin().y == v.origin().y);
      for (int k = 0; k < want[2]; ++k)
        for (int j = 0; j < want[1]; ++j)
          for (int i = 0; i < want[0]; ++i) {
            double best = -std::numeric_limits<double>::infinity();
            for (int t = 0; t < v.dims()[axis]; ++t)
              best = std::max(best, v.at(axis == 0 ? t : i, axis == 1 ? t : j, axis == 2 ? t : k));
            CHECK(m.at(i, j, k) == best);
          }
    }
    CHECK_THROWS(post::mip(v, 3));
    CHECK_THROWS(post::mip(v, -1));
  });

  run("psnr follows the inverse-mse law; identical images score perfectly", [&] {
    VoxelGrid a({16, 1, 16}, {1, 1, 1}, {0, 0, 0}), b = a;
    std::mt19937 rng(21);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (std::size_t i = 0; i < a.data().size(); ++i) {
      a.data()[i] = u(rng);
      b.data()[i] = std::clamp(a.data()[i] + 0.05 * (u(rng) - 0.5), 0.0, 1.0);
    }
    post::MetricsReport r = post::metrics(a, b);
    double sq = 0.0;
    for (std::size_t i = 0; i < a.data().size(); ++i)
      sq += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
    CHECK(std::abs(r.mse - sq / a.data().size()) <= 1e-12 * r.mse);
    CHECK(std::abs(r.psnr - 10.0 * std::log10(1.0 / r.mse)) <= 1e-12);
    CHECK(r.ssim < 1.0 && r.ssim > -1.0);
    post::MetricsReport same = post::metrics(a, a);
    CHECK(same.mse == 0.0 && std::isinf(same.psnr) && same.psnr > 0.0 && same.ssim == 1.0);
    VoxelGrid c({16, 16, 1}, {1, 1, 1}, {0, 0, 0});
    CHECK_THROWS(post::metrics(a, c));
  });

  run("ground truth perfusion image is a peak-normalised splat", [&] {
    auto g = grid3(9, 9, 9);
    std::vector<std::vector<Vec3>> tracks(2);
    Vec3 c0 = g.point(4 + 9 * (4 + 9 * 4));
    tracks[0].push_back(c0);
    tracks[1].push_back(c0);
    VoxelGrid gt = post::ground_truth_pd(tracks, g, 1.0);
    CHECK(gt.at(4, 4, 4) == 1.0);
    CHECK(std::abs(gt.at(5, 4, 4) - std::exp(-0.5)) <= 1e-12);
    CHECK(gt.at(0, 0, 0) == 0.0);  // beyond three sigma
    CHECK_THROWS(post::ground_truth_pd({}, g, 1.0));
    CHECK_THROWS(post::ground_truth_pd(tracks, g, 0.0));
  });

  // ---- RF synthesis (test_rf.cpp:312-594), now on the GPU ----
  auto rf_probe = [](int n, int v, double fc, double bw) {
    Transducer t;
    t.name = "test";
    t.pitch = 0.4e-3;
    t.half_width = 0.15e-3;
    t.subelements = v;
    t.center_frequency = fc;
    t.fractional_bandwidth = bw;
    for (int i = 0; i < n; ++i) t.elements.push_back({(i - (n - 1) / 2.0) * t.pitch, 0.0, 0.0});
    return t;
  };
  run("doubling reflectivity doubles every rf sample exactly; blocks change nothing", [&] {
    Transducer td = rf_probe(5, 2, 5e6, 0.5);
    TxEvent tx = rf::plane_wave_delays(td, 2.0 * kPi / 180.0, 1540.0);
    rf::MediumParams med;
    std::mt19937 rng(11);
    std::uniform_real_distribution<double> ux(-2e-3, 2e-3), uz(6e-3, 14e-3);
    std::normal_distribution<double> nd(0.0, 1.0);
    tissue::ScattererCloud cloud;
    for (int i = 0; i < 200; ++i) {
      cloud.positions.push_back({ux(rng), 0.0, uz(rng)});
      cloud.reflectivity.push_back(nd(rng));
    }
    tissue::ScattererCloud doubled = cloud;
    for (double& r : doubled.reflectivity) r *= 2.0;
    rf::RfSimStats st;
    RfFrame base = rf::simulate_rf(cloud, td, tx, med, 20e6, 25e-6, &st);
    RfFrame twice = rf::simulate_rf(doubled, td, tx, med, 20e6, 25e-6);
    CHECK(base.n_samples == 500 && base.n_elements == 5 && st.blocks == 1);
    CHECK(st.pair_bin_products == 200ull * 10 * st.frequencies);
    for (std::size_t i = 0; i < base.samples.size(); ++i) CHECK(twice.samples[i] == 2.0 * base.samples[i]);
    rf::RfChunkPlan probe = rf::plan_rf_chunks(td, 200, med, 20e6, 25e-6, SIZE_MAX);
    std::size_t budget = probe.fixed_bytes + 50 * probe.per_scatterer_bytes;
    rf::RfSimStats st4;
    RfFrame ch = rf::simulate_rf_chunked(cloud, td, tx, med, 20e6, 25e-6, budget, &st4);
    CHECK(st4.blocks == 4 && st4.peak_tracked_bytes <= budget);
    for (std::size_t i = 0; i < base.samples.size(); ++i) CHECK(ch.samples[i] == base.samples[i]);
  });

  run("rf composition adds exactly; frames round-trip through the container", [&] {
    Transducer td = rf_probe(4, 2, 5e6, 0.5);
    TxEvent tx = rf::plane_wave_delays(td, 0.0, 1540.0);
    rf::MediumParams med;
    tissue::ScattererCloud tis, flow;
    tis.positions = {{0.3e-3, 0.0, 8e-3}, {-0.5e-3, 0.0, 11e-3}};
    tis.reflectivity = {1.0, -0.4};
    flow.positions = {{0.0, 0.0, 9.5e-3}};
    flow.reflectivity = {0.1};
    rf::ComposeStats cs;
    auto totals = rf::compose_frames({tis}, {flow, flow}, true, td, tx, med, 20e6, 25e-6, &cs);
    CHECK(cs.tissue_simulations == 1 && cs.flow_simulations == 2 && totals.size() == 2);
    RfFrame a = rf::simulate_rf(tis, td, tx, med, 20e6, 25e-6);
    RfFrame b = rf::simulate_rf(flow, td, tx, med, 20e6, 25e-6);
    for (std::size_t i = 0; i < a.samples.size(); ++i) CHECK(totals[1].samples[i] == a.samples[i] + b.samples[i]);
    auto dir = std::filesystem::temp_directory_path() / "fqf_dropin_rf";
    std::filesystem::create_directories(dir);
    rf::write_rf_frame((dir / "f.fqf").string(), a, 7);
    auto [back, idx] = rf::read_rf_frame((dir / "f.fqf").string());
    CHECK(idx == 7 && back.n_samples == a.n_samples && back.n_elements == a.n_elements);
    for (std::size_t i = 0; i < a.samples.size(); ++i)
      CHECK(back.samples[i] == static_cast<double>(static_cast<float>(a.samples[i])));
  });

  run("rf input contract violations throw", [&] {
    Transducer td = rf_probe(3, 2, 5e6, 0.5);
    TxEvent tx = rf::plane_wave_delays(td, 0.0, 1540.0);
    rf::MediumParams med;
    tissue::ScattererCloud cloud;
    cloud.positions = {{0.0, 0.0, 9e-3}};
    cloud.reflectivity = {1.0};
    CHECK_THROWS(rf::simulate_rf(cloud, td, tx, med, 19e6, 20e-6));
    rf::MediumParams relaxed = med;
    relaxed.min_fs_ratio = 2.0;
    CHECK(rf::simulate_rf(cloud, td, tx, relaxed, 19e6, 20e-6).n_samples == 380);
    tissue::ScattererCloud deep;
    deep.positions = {{0.0, 0.0, 20e-3}};
    deep.reflectivity = {1.0};
    CHECK_THROWS(rf::simulate_rf(deep, td, tx, med, 20e6, 20e-6));
    tissue::ScattererCloud bad = cloud;
    bad.positions[0].z = std::numeric_limits<double>::quiet_NaN();
    CHECK_THROWS(rf::simulate_rf(bad, td, tx, med, 20e6, 20e-6));
    CHECK_THROWS(rf::simulate_rf(tissue::ScattererCloud{}, td, tx, med, 20e6, 20e-6));
    TxEvent short_tx = tx;
    short_tx.delays.pop_back();
    CHECK_THROWS(rf::simulate_rf(cloud, td, short_tx, med, 20e6, 20e-6));
  });

  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
