// fqf_stages.cpp -- run_beamform + run_post (proj/src/pipeline/run.cpp:397-487)
// as one C++ stage body over the reconstruction engine (fqfg_recon_*): RF
// frames -> demodulation + DAS + Casorati filter + power Doppler with the IQ
// ensemble resident in HBM, then the reference's stage outputs.
//
// File formats are the reference's own functions where the drop-in library
// provides them (rf::read_rf_frame, beamform::write_iq_volume, write_grid,
// post::write_pgm, post::bmode / render_db / mip / ground_truth_pd on the
// GPU); the particle container (hemo/particles.cpp:81-95) is read through the
// reference's container API, and svd_report.json restates nlohmann's
// dump(2) (run.cpp:470-485; the vendored json.hpp is absent) -- the Python
// stage bodies (paper_2509_05464_b200/stages.py) write the same bytes.
#include "fqf_stages.hpp"

#include <charconv>
#include <cmath>
#include <complex>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "fqf/core/container.hpp"
#include "fqf/core/error.hpp"
#include "fqf/core/grid.hpp"
#include "fqf/post/render.hpp"
#include "fqf/rf/simulate.hpp"
#include "fqfgpu.h"

namespace fs = std::filesystem;

namespace fqf::gpu {
namespace {

void ok(int rc) {
  if (rc != FQFG_OK) throw Error(fqfg_last_error());
}

std::string rf_frame_rel(int f, int a) {  // run.cpp:86-88
  char b[64];
  std::snprintf(b, sizeof b, "rf/frame_%04d_tx_%02d.fqf", f, a);
  return b;
}
std::string iq_frame_rel(int f) { return "beamform/Frame_" + std::to_string(f + 1) + ".fqf"; }
std::string particle_frame_rel(int f) {  // run.cpp:84
  char b[64];
  std::snprintf(b, sizeof b, "particles/frame_%04d.fqf", f);
  return b;
}

// hemo::read_particle_frame (particles.cpp:81-95): positions only.
std::vector<Vec3> read_particles(const std::string& path) {
  auto [header, payload] = read_container(path);
  require(find_header(header, "kind") && header_value(header, "kind") == "particles", path,
          ": not a particle container");
  std::vector<double> flat = as_real_f64(payload);
  require(flat.size() % 3 == 0, path, ": particle payload is not 3 doubles per point");
  std::vector<Vec3> p(flat.size() / 3);
  for (std::size_t i = 0; i < p.size(); ++i) p[i] = {flat[3 * i], flat[3 * i + 1], flat[3 * i + 2]};
  return p;
}

// nlohmann::json's double output: the shortest round-trip digits
// (std::to_chars), fixed notation for decimal exponents in (-4, 15], '.0' on
// integral values, else d.ddde+XX; non-finite -> null.
std::string json_number(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof buf, std::fabs(x), std::chars_format::scientific);
  std::string sci(buf, res.ptr);  // d[.ddd]e[+-]XX
  const auto epos = sci.find('e');
  std::string digits = sci.substr(0, 1) + (epos > 2 ? sci.substr(2, epos - 2) : "");
  const int e10 = std::stoi(sci.substr(epos + 1));
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = (int)digits.size(), n = e10 + 1;  // value = 0.DIGITS x 10^n
  std::string s;
  if (k <= n && n <= 15) {
    s = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    s = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    s = "0." + std::string(-n, '0') + digits;
  } else {
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "%s%02d", e >= 0 ? "e+" : "e-", e >= 0 ? e : -e);
    s = digits.substr(0, 1) + (k > 1 ? "." + digits.substr(1) : "") + eb;
  }
  return (x < 0 ? "-" : "") + s;
}

// run.cpp:470-482: nlohmann object (keys sorted), dump(2) + newline.
std::string svd_report_json(const std::vector<double>& sigma, const std::vector<double>& corr,
                            int lo, int hi) {
  auto arr = [](const std::vector<std::string>& xs) {
    if (xs.empty()) return std::string("[]");
    std::string s = "[\n";
    for (std::size_t i = 0; i < xs.size(); ++i) s += "    " + xs[i] + (i + 1 < xs.size() ? ",\n" : "\n");
    return s + "  ]";
  };
  std::vector<std::string> c, sg;
  for (double v : corr) c.push_back(json_number(v));
  for (double v : sigma) sg.push_back(json_number(v));
  std::ostringstream os;
  os << "{\n  \"keep\": " << arr({std::to_string(lo), std::to_string(hi)})
     << ",\n  \"mode_correlation\": " << arr(c) << ",\n  \"n_modes\": " << sigma.size()
     << ",\n  \"singular_values\": " << arr(sg) << "\n}\n";
  return os.str();
}

struct Engine {
  fqfg_recon R = nullptr;
  ~Engine() { fqfg_recon_destroy(R); }
};

}  // namespace

std::vector<std::string> run_beamform_post(const std::string& out, const StageConfig& cfg,
                                           bool write_frames) {
  const int F = cfg.n_frames, A = (int)cfg.angles_deg.size();
  require(F >= 1 && A >= 1, "stage needs at least one frame and one transmit");
  // ---- beamform inputs (run.cpp:398-410): RF frames, header checks.
  int T = 0, E = 0;
  double fs = 0.0;
  std::vector<double> t0(A, 0.0), angles(A, 0.0);
  std::vector<float> rf;
  for (int f = 0; f < F; ++f)
    for (int a = 0; a < A; ++a) {
      const fs::path p = fs::path(out) / rf_frame_rel(f, a);
      auto [frame, index] = rf::read_rf_frame(p.string());
      require(index == f, p.string(), ": header frame index ", index, " does not match ", f);
      if (f == 0 && a == 0) {
        T = frame.n_samples, E = frame.n_elements, fs = frame.sampling_rate;
        rf.resize((std::size_t)F * A * T * E);
      }
      require(frame.n_samples == T && frame.n_elements == E && frame.sampling_rate == fs,
              "frames of an ensemble must share the recording shape and sampling rate");
      if (f == 0) t0[a] = frame.t0, angles[a] = frame.tx.angle;
      require(frame.t0 == t0[a] && frame.tx.angle == angles[a],
              "transmit slot ", a, " changes its start time or angle across frames");
      float* dst = rf.data() + ((std::size_t)f * A + a) * T * E;
      for (std::size_t i = 0; i < frame.samples.size(); ++i) dst[i] = (float)frame.samples[i];
    }
  // ---- one engine pass: RF -> IQ (resident) -> filter -> PD.
  const int hi = cfg.svd_hi == 0 ? F : cfg.svd_hi;
  fqfg_rf_desc desc{F, A, T, E, fs, t0.data(), angles.data()};
  const beamform::GridSpec& g = cfg.grid;
  fqfg_grid grid{{g.dims[0], g.dims[1], g.dims[2]},
                 {g.spacing.x, g.spacing.y, g.spacing.z},
                 {g.origin.x, g.origin.y, g.origin.z}};
  std::vector<double> el;
  for (const Vec3& e : cfg.transducer.elements) el.insert(el.end(), {e.x, e.y, e.z});
  fqfg_probe probe{(int)cfg.transducer.elements.size(), el.data()};
  fqfg_bf bf{cfg.sound_speed, cfg.transducer.center_frequency, cfg.f_number, 1, cfg.lowpass_taps};
  fqfg_recon_opts opts{};
  opts.keep_lo = cfg.svd_lo;
  opts.keep_hi = hi;
  opts.world = 1;
  Engine eng;
  ok(fqfg_recon_create(&desc, &grid, &probe, &bf, &opts, &eng.R));
  const std::size_t N = g.num_points();
  std::vector<double> pd(N);
  const float* rfs[1] = {rf.data()};
  double* pds[1] = {pd.data()};
  ok(fqfg_recon_run(eng.R, 1, rfs, pds, nullptr));
  std::vector<double> sigma(F), corr((std::size_t)F * F);
  ok(fqfg_recon_report(eng.R, sigma.data(), corr.data()));

  std::vector<std::string> outputs;
  // ---- beamform outputs (run.cpp:425-430): the F IQ volumes.
  std::vector<std::complex<float>> iq((std::size_t)F * N);
  ok(fqfg_recon_copy_iq(eng.R, 0, N, reinterpret_cast<float*>(iq.data())));
  auto volume = [&](int f) {
    beamform::IqVolume v;
    v.grid = g;
    v.frame_index = f;
    v.n_angles = A;
    v.values.resize(N);
    for (std::size_t i = 0; i < N; ++i) v.values[i] = std::complex<double>(iq[(std::size_t)f * N + i]);
    return v;
  };
  if (write_frames) {
    fs::create_directories(fs::path(out) / "beamform");
    for (int f = 0; f < F; ++f) {
      beamform::write_iq_volume((fs::path(out) / iq_frame_rel(f)).string(), volume(f));
      outputs.push_back(iq_frame_rel(f));
    }
  }
  // ---- post outputs (run.cpp:441-486).
  fs::create_directories(fs::path(out) / "post");
  auto save_image = [&](const VoxelGrid& img, const std::string& stem) {
    write_grid((fs::path(out) / ("post/" + stem + ".fqf")).string(), img);
    outputs.push_back("post/" + stem + ".fqf");
    const auto& d = img.dims();
    VoxelGrid flat = (d[0] == 1 || d[1] == 1 || d[2] == 1) ? img : post::mip(img, 1);
    post::write_pgm((fs::path(out) / ("post/" + stem + ".pgm")).string(), flat);
    outputs.push_back("post/" + stem + ".pgm");
  };
  save_image(post::bmode(volume(0), cfg.bmode_dynamic_range_db), "bmode");
  VoxelGrid pdg(g.dims, g.spacing, g.origin);
  std::copy(pd.begin(), pd.end(), pdg.data().begin());
  save_image(post::render_db(pdg, cfg.pd_dynamic_range_db, post::DbScale::power), "pd");
  std::vector<std::vector<Vec3>> tracks(F);
  for (int f = 0; f < F; ++f) tracks[f] = read_particles((fs::path(out) / particle_frame_rel(f)).string());
  VoxelGrid gt = post::ground_truth_pd(tracks, g, cfg.ground_truth_sigma_voxels);
  save_image(post::render_db(gt, cfg.pd_dynamic_range_db, post::DbScale::power), "gt");
  {
    const fs::path p = fs::path(out) / "post/svd_report.json";
    std::ofstream f(p);
    f << svd_report_json(sigma, corr, cfg.svd_lo, hi);
    require(f.good(), "cannot write ", p.string());
    outputs.push_back("post/svd_report.json");
  }
  return outputs;
}

}  // namespace fqf::gpu

// C entry for bindings and tests: the StageConfig as "key=value" lines
// (n_frames, angles_deg, sound_speed, f_number, lowpass_taps, dims,
// spacing, origin, center_frequency, elements (3 E numbers), bmode_dr, pd_dr,
// svd_lo, svd_hi, gt_sigma, write_frames).  Returns 0 or FQFG_EINVAL with the
// message in fqfg_stage_last_error().
namespace {
thread_local std::string g_stage_err;
}

extern "C" __attribute__((visibility("default"))) const char* fqfg_stage_last_error(void) {
  return g_stage_err.c_str();
}

extern "C" __attribute__((visibility("default"))) int fqfg_stage_beamform_post(const char* out,
                                                                               const char* cfg_text) {
  try {
    fqf::gpu::StageConfig c;
    bool write_frames = true;
    std::istringstream in(cfg_text);
    std::string line;
    auto nums = [](const std::string& s) {
      std::vector<double> v;
      std::istringstream is(s);
      double x;
      while (is >> x) v.push_back(x);
      return v;
    };
    while (std::getline(in, line)) {
      const auto eq = line.find('=');
      if (eq == std::string::npos) continue;
      const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
      const std::vector<double> n = nums(v);
      if (k == "n_frames") c.n_frames = (int)n.at(0);
      else if (k == "angles_deg") c.angles_deg = n;
      else if (k == "sound_speed") c.sound_speed = n.at(0);
      else if (k == "f_number") c.f_number = n.at(0);
      else if (k == "lowpass_taps") c.lowpass_taps = (int)n.at(0);
      else if (k == "dims") c.grid.dims = {(int)n.at(0), (int)n.at(1), (int)n.at(2)};
      else if (k == "spacing") c.grid.spacing = {n.at(0), n.at(1), n.at(2)};
      else if (k == "origin") c.grid.origin = {n.at(0), n.at(1), n.at(2)};
      else if (k == "center_frequency") c.transducer.center_frequency = n.at(0);
      else if (k == "elements") {
        c.transducer.elements.clear();
        for (std::size_t i = 0; i + 2 < n.size(); i += 3) c.transducer.elements.push_back({n[i], n[i + 1], n[i + 2]});
      } else if (k == "bmode_dr") c.bmode_dynamic_range_db = n.at(0);
      else if (k == "pd_dr") c.pd_dynamic_range_db = n.at(0);
      else if (k == "svd_lo") c.svd_lo = (int)n.at(0);
      else if (k == "svd_hi") c.svd_hi = (int)n.at(0);
      else if (k == "gt_sigma") c.ground_truth_sigma_voxels = n.at(0);
      else if (k == "write_frames") write_frames = n.at(0) != 0.0;
    }
    fqf::gpu::run_beamform_post(out, c, write_frames);
    return 0;
  } catch (const std::exception& e) {
    g_stage_err = e.what();
    return FQFG_EINVAL;
  }
}
