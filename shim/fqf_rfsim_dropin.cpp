// fqf_rfsim_dropin.cpp -- the reference's RF simulator API (rf/simulate.hpp)
// over the B200 C ABI (include/fqfgpu.h, csrc/rfsim.cu).
//
// Compiled against the reference's own headers, so every signature is the
// reference's by construction.  It replaces proj/src/rf/simulate.cpp in a
// libfqf build -- which also drops the FFTW dependency (simulate.cpp:3).
// The simulation runs on the GPU; this file marshals the scatterer cloud and
// transmit event, turns a nonzero status into fqf::Error(fqfg_last_error()),
// and keeps the reference's composition and container I/O semantics.
#include <cmath>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "fqf/core/container.hpp"
#include "fqf/core/error.hpp"
#include "fqf/rf/simulate.hpp"
#include "fqf/rf/transducer.hpp"
#include "fqfgpu.h"

namespace fqf::rf {
namespace {

void ok(int rc) {
  if (rc != FQFG_OK) throw Error(fqfg_last_error());
}

struct CTransducer {
  std::vector<double> xyz;
  fqfg_transducer t{};
  explicit CTransducer(const Transducer& td) {
    for (const Vec3& e : td.elements) xyz.insert(xyz.end(), {e.x, e.y, e.z});
    t.n_elements = td.n_elements();
    t.xyz = xyz.data();
    t.half_width = td.half_width;
    t.subelements = td.subelements;
    t.pitch = td.pitch;
    t.center_frequency = td.center_frequency;
    t.fractional_bandwidth = td.fractional_bandwidth;
    t.elevation_height = td.elevation_height;
    t.elevation_focus = td.elevation_focus;
    t.elevation_core_weight = td.elevation_core_weight;
    t.elevation_tail_weight = td.elevation_tail_weight;
    t.elevation_aperture_factor = td.elevation_aperture_factor;
  }
};

fqfg_medium c_medium(const MediumParams& m) {
  return fqfg_medium{m.c, m.attenuation_db_cm_mhz, m.scatterer_memory_budget, m.min_fs_ratio};
}

RfFrame run(const tissue::ScattererCloud& cloud, const Transducer& t, const TxEvent& tx,
            const MediumParams& medium, double fs, double duration, int chunked,
            std::size_t budget, RfSimStats* stats) {
  validate_transducer(t);
  require(!cloud.positions.empty(), "scatterer cloud is empty");
  require(cloud.reflectivity.size() == cloud.positions.size(),
          "cloud reflectivity count does not match positions");
  require(tx.delays.size() == t.elements.size(), "transmit delays do not match element count");
  require(tx.apodization.size() == t.elements.size(),
          "transmit apodization does not match element count");
  std::vector<double> pos;
  pos.reserve(cloud.positions.size() * 3);
  for (const Vec3& p : cloud.positions) pos.insert(pos.end(), {p.x, p.y, p.z});
  CTransducer ct(t);
  fqfg_medium m = c_medium(medium);
  const int T = std::max(16, static_cast<int>(std::llround(fs * duration)));
  std::vector<double> out(static_cast<std::size_t>(T) * t.elements.size());
  int n = 0;
  fqfg_rfsim_stats st{};
  ok(fqfg_simulate_rf(pos.data(), cloud.reflectivity.data(), cloud.positions.size(), &ct.t,
                      tx.delays.data(), tx.apodization.data(), &m, fs, duration, chunked, budget,
                      out.data(), &n, &st));
  RfFrame frame;
  frame.n_samples = n;
  frame.n_elements = t.n_elements();
  frame.sampling_rate = fs;
  frame.t0 = 0.0;
  frame.tx = tx;
  out.resize(static_cast<std::size_t>(n) * t.elements.size());
  frame.samples = std::move(out);
  if (stats) {
    stats->blocks = st.blocks;
    stats->frequencies = st.frequencies;
    stats->peak_tracked_bytes = st.peak_tracked_bytes;
    stats->pair_bin_products = st.pair_bin_products;
  }
  return frame;
}

std::string fmt17(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

}  // namespace

RfChunkPlan plan_rf_chunks(const Transducer& t, std::size_t n_scatterers,
                           const MediumParams& medium, double sampling_rate, double duration,
                           std::size_t budget) {
  validate_transducer(t);
  CTransducer ct(t);
  fqfg_medium m = c_medium(medium);
  fqfg_rf_chunk_plan p{};
  ok(fqfg_plan_rf_chunks(&ct.t, n_scatterers, &m, sampling_rate, duration, budget, &p));
  RfChunkPlan plan;
  plan.blocks = p.blocks;
  plan.block_scatterers = p.block_scatterers;
  plan.per_scatterer_bytes = p.per_scatterer_bytes;
  plan.fixed_bytes = p.fixed_bytes;
  return plan;
}

RfFrame simulate_rf(const tissue::ScattererCloud& cloud, const Transducer& t, const TxEvent& tx,
                    const MediumParams& medium, double sampling_rate, double duration,
                    RfSimStats* stats) {
  return run(cloud, t, tx, medium, sampling_rate, duration, 0, 0, stats);
}

RfFrame simulate_rf_chunked(const tissue::ScattererCloud& cloud, const Transducer& t,
                            const TxEvent& tx, const MediumParams& medium, double sampling_rate,
                            double duration, std::size_t budget, RfSimStats* stats) {
  return run(cloud, t, tx, medium, sampling_rate, duration, 1, budget, stats);
}

// simulate.cpp:608-644 semantics: tissue echoes (once if static) plus flow
// echoes per frame, empty clouds contribute zero frames.
std::vector<RfFrame> compose_frames(const std::vector<tissue::ScattererCloud>& tissue_frames,
                                    const std::vector<tissue::ScattererCloud>& flow_frames,
                                    bool static_tissue, const Transducer& t, const TxEvent& tx,
                                    const MediumParams& medium, double sampling_rate,
                                    double duration, ComposeStats* stats) {
  require(!flow_frames.empty(), "no flow frames to compose");
  if (static_tissue) {
    require(!tissue_frames.empty(), "static tissue requires one tissue cloud");
  } else {
    require(tissue_frames.size() == flow_frames.size(),
            "tissue and flow frame counts do not match");
  }
  ComposeStats local;
  auto sim = [&](const tissue::ScattererCloud& cloud, int& counter) {
    if (cloud.positions.empty()) {
      validate_transducer(t);
      RfFrame z;
      z.n_samples = static_cast<int>(std::llround(sampling_rate * duration));
      z.n_elements = t.n_elements();
      z.sampling_rate = sampling_rate;
      z.tx = tx;
      z.samples.assign(static_cast<std::size_t>(z.n_samples) * t.elements.size(), 0.0);
      return z;
    }
    ++counter;
    return simulate_rf_chunked(cloud, t, tx, medium, sampling_rate, duration,
                               medium.scatterer_memory_budget);
  };
  std::vector<RfFrame> out;
  out.reserve(flow_frames.size());
  RfFrame tissue_rf;
  if (static_tissue) tissue_rf = sim(tissue_frames[0], local.tissue_simulations);
  for (std::size_t i = 0; i < flow_frames.size(); ++i) {
    if (!static_tissue) tissue_rf = sim(tissue_frames[i], local.tissue_simulations);
    RfFrame flow_rf = sim(flow_frames[i], local.flow_simulations);
    RfFrame total = tissue_rf;
    for (std::size_t k = 0; k < total.samples.size(); ++k) total.samples[k] += flow_rf.samples[k];
    out.push_back(std::move(total));
  }
  if (stats) *stats = local;
  return out;
}

// FQF1 "rf" containers (f32 payload, time-major), via the reference's
// container API.
void write_rf_frame(const std::string& path, const RfFrame& frame, int frame_index) {
  ContainerHeader h;
  h.emplace_back("kind", "rf");
  h.emplace_back("samples", std::to_string(frame.n_samples));
  h.emplace_back("elements", std::to_string(frame.n_elements));
  h.emplace_back("sampling_rate", fmt17(frame.sampling_rate));
  h.emplace_back("t0", fmt17(frame.t0));
  h.emplace_back("angle", fmt17(frame.tx.angle));
  h.emplace_back("frame", std::to_string(frame_index));
  std::vector<float> f32(frame.samples.begin(), frame.samples.end());
  write_container(path, h, make_payload(std::span<const float>(f32)));
}

std::pair<RfFrame, int> read_rf_frame(const std::string& path) {
  auto [header, payload] = read_container(path);
  require(find_header(header, "kind") && header_value(header, "kind") == "rf", path,
          ": not an rf frame container");
  RfFrame frame;
  frame.n_samples = std::stoi(header_value(header, "samples"));
  frame.n_elements = std::stoi(header_value(header, "elements"));
  frame.sampling_rate = std::stod(header_value(header, "sampling_rate"));
  frame.t0 = std::stod(header_value(header, "t0"));
  frame.tx.angle = std::stod(header_value(header, "angle"));
  int index = std::stoi(header_value(header, "frame"));
  frame.samples = as_real_f64(payload);
  require(frame.samples.size() ==
              static_cast<std::size_t>(frame.n_samples) * static_cast<std::size_t>(frame.n_elements),
          path, ": sample count does not match header dimensions");
  return {std::move(frame), index};
}

}  // namespace fqf::rf
