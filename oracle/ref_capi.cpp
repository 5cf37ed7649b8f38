// ref_capi.cpp -- C-ABI wrapper over the REFERENCE's own, unmodified sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's proj/src/{core/*,rf/transducer,beamform/{iq,das},
// post/{render,metrics}}.cpp straight from /root/reference into
// oracle/_ref/libfqf_ref.so (git-ignored).  No reference source is copied into
// this repository.  It is used to pin the C restatement (fqf_oracle.c), to
// generate tests/golden/, and as bench.py's `--impl reference` CPU arm.
//
// svd_filter (post/svd.cpp) needs Eigen, which is absent from this image, so
// it is not wrapped; the restatement in fqf_oracle.c stands in for it.
#include <complex>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#include "fqf/beamform/das.hpp"
#include "fqf/core/grid.hpp"
#include "fqf/beamform/iq.hpp"
#include "fqf/core/error.hpp"
#include "fqf/post/metrics.hpp"
#include "fqf/post/render.hpp"
#include "fqf/rf/simulate.hpp"
#include "fqf/rf/transducer.hpp"

using namespace fqf;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

rf::Transducer make_probe(int E, const double* xyz, double fc) {
  rf::Transducer t;
  t.name = "capi";
  t.pitch = 0.3e-3;
  t.half_width = 0.135e-3;
  t.subelements = 2;
  t.center_frequency = fc > 0 ? fc : 1.0;
  t.fractional_bandwidth = 0.6;
  t.elevation_height = 0.0;
  for (int e = 0; e < E; ++e) t.elements.push_back({xyz[3 * e], xyz[3 * e + 1], xyz[3 * e + 2]});
  return t;
}

beamform::GridSpec make_grid(const int* dims, const double* sp, const double* org) {
  beamform::GridSpec g;
  g.dims = {dims[0], dims[1], dims[2]};
  g.spacing = {sp[0], sp[1], sp[2]};
  g.origin = {org[0], org[1], org[2]};
  return g;
}
rf::Transducer make_sim_probe(int E, const double* xyz, int subelements, const double* tp) {
  rf::Transducer td;
  td.name = "capi";
  for (int e = 0; e < E; ++e) td.elements.push_back({xyz[3 * e], xyz[3 * e + 1], xyz[3 * e + 2]});
  td.half_width = tp[0];
  td.subelements = subelements;
  td.pitch = tp[1];
  td.center_frequency = tp[2];
  td.fractional_bandwidth = tp[3];
  td.elevation_height = tp[4];
  td.elevation_focus = tp[5];
  td.elevation_core_weight = tp[6];
  td.elevation_tail_weight = tp[7];
  td.elevation_aperture_factor = tp[8];
  return td;
}

tissue::ScattererCloud make_cloud(const double* pos, const double* refl, std::size_t n) {
  tissue::ScattererCloud c;
  for (std::size_t i = 0; i < n; ++i) {
    c.positions.push_back({pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]});
    c.reflectivity.push_back(refl[i]);
    c.label.push_back(tissue::Label{});
  }
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// The reference tests draw their inputs from libstdc++ engines
// (test_beamform.cpp: std::mt19937 + uniform_real_distribution(-1, 1);
// test_post.cpp: std::mt19937_64 + normal_distribution).  One distribution
// object per call, values in draw order, so a caller can replay any fixture.
void ref_mt19937_uniform(std::uint32_t seed, std::size_t n, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void ref_mt19937_64_normal(std::uint64_t seed, std::size_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd;
  for (std::size_t i = 0; i < n; ++i) out[i] = nd(rng);
}

int ref_rf_to_iq(const double* rf, int T, int E, double fs, double t0, double fc, int taps,
                 double* iq) {
  return guarded([&] {
    rf::RfFrame f;
    f.n_samples = T;
    f.n_elements = E;
    f.sampling_rate = fs;
    f.t0 = t0;
    f.samples.assign(rf, rf + static_cast<std::size_t>(T) * E);
    beamform::IqFrame out = beamform::rf_to_iq(f, fc, taps);
    std::memcpy(iq, out.samples.data(), out.samples.size() * sizeof(std::complex<double>));
  });
}

long ref_plan_chunks(std::size_t n, int a, std::size_t budget, std::size_t* ranges) {
  long k = -1;
  int rc = guarded([&] {
    beamform::ChunkPlan p = beamform::plan_chunks(n, a, budget);
    k = p.n_chunks;
    if (ranges)
      for (int i = 0; i < p.n_chunks; ++i) {
        ranges[2 * i] = p.ranges[i].first;
        ranges[2 * i + 1] = p.ranges[i].second;
      }
  });
  return rc ? -1 : k;
}

// stats_out: chunks, matrix_builds, out_of_window, matrix_bytes_peak,
// accumulator_bytes_peak.  opts: memory_budget, matrix_budget, cache (0/1).
int ref_das(const double* rf, int F, int A, int T, int E, double fs, const double* t0,
            const double* angles, const double* elements, const int* dims, const double* spacing,
            const double* origin, double c, double fc, double f_number, int interp, int taps,
            std::size_t mem_budget, std::size_t matrix_budget, int cache, double* iq_out,
            std::uint64_t* stats_out) {
  return guarded([&] {
    rf::Transducer td = make_probe(E, elements, fc);
    beamform::GridSpec grid = make_grid(dims, spacing, origin);
    std::vector<std::vector<rf::RfFrame>> frames(F);
    for (int f = 0; f < F; ++f)
      for (int a = 0; a < A; ++a) {
        rf::RfFrame fr;
        fr.n_samples = T;
        fr.n_elements = E;
        fr.sampling_rate = fs;
        fr.t0 = t0[a];
        fr.tx.angle = angles[a];
        const double* src = rf + (static_cast<std::size_t>(f) * A + a) * T * E;
        fr.samples.assign(src, src + static_cast<std::size_t>(T) * E);
        frames[f].push_back(std::move(fr));
      }
    beamform::BeamformParams bp;
    bp.c = c;
    bp.center_frequency = fc;
    bp.f_number = f_number;
    bp.interp_order = interp;
    bp.lowpass_taps = taps;
    beamform::DasOptions opts;
    opts.memory_budget_bytes = mem_budget;
    opts.matrix_budget_bytes = matrix_budget;
    opts.cache_matrices = cache != 0;
    beamform::DasStats st;
    std::vector<beamform::IqVolume> vols = beamform::das_reconstruct(frames, grid, td, bp, opts, &st);
    std::size_t n = grid.num_points();
    for (int f = 0; f < F; ++f)
      std::memcpy(iq_out + 2 * static_cast<std::size_t>(f) * n, vols[f].values.data(),
                  n * sizeof(std::complex<double>));
    if (stats_out) {
      stats_out[0] = st.chunks;
      stats_out[1] = st.matrix_builds;
      stats_out[2] = st.out_of_window;
      stats_out[3] = st.matrix_bytes_peak;
      stats_out[4] = st.accumulator_bytes_peak;
    }
  });
}

int ref_power_doppler(const double* iq, int F, const int* dims, double* pd) {
  return guarded([&] {
    beamform::GridSpec g;
    g.dims = {dims[0], dims[1], dims[2]};
    std::size_t n = g.num_points();
    std::vector<beamform::IqVolume> ens(F);
    for (int f = 0; f < F; ++f) {
      ens[f].grid = g;
      ens[f].frame_index = f;
      const auto* src = reinterpret_cast<const std::complex<double>*>(iq) + f * n;
      ens[f].values.assign(src, src + n);
    }
    VoxelGrid out = post::power_doppler(ens);
    std::memcpy(pd, out.data().data(), n * sizeof(double));
  });
}

// scale: 0 = amplitude (20 log10), 1 = power (10 log10).
int ref_render_db(const double* vol, const int* dims, double dr_db, int scale, double* out) {
  return guarded([&] {
    VoxelGrid g({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    std::memcpy(g.data().data(), vol, g.data().size() * sizeof(double));
    VoxelGrid r = post::render_db(g, dr_db, scale ? post::DbScale::power : post::DbScale::amplitude);
    std::memcpy(out, r.data().data(), r.data().size() * sizeof(double));
  });
}

int ref_metrics(const double* test, const double* refimg, const int* dims, double* mse_psnr_ssim) {
  return guarded([&] {
    VoxelGrid a({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    VoxelGrid b({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    std::memcpy(a.data().data(), test, a.data().size() * sizeof(double));
    std::memcpy(b.data().data(), refimg, b.data().size() * sizeof(double));
    post::MetricsReport m = post::metrics(a, b);
    mse_psnr_ssim[0] = m.mse;
    mse_psnr_ssim[1] = m.psnr;
    mse_psnr_ssim[2] = m.ssim;
  });
}

// bmode (render.cpp:70-78): iq [N][2] complex<double>.
int ref_bmode(const double* iq, const int* dims, double dr_db, double* out) {
  return guarded([&] {
    beamform::IqVolume v;
    v.grid.dims = {dims[0], dims[1], dims[2]};
    std::size_t n = v.grid.num_points();
    const auto* src = reinterpret_cast<const std::complex<double>*>(iq);
    v.values.assign(src, src + n);
    VoxelGrid r = post::bmode(v, dr_db);
    std::memcpy(out, r.data().data(), n * sizeof(double));
  });
}

// mip (render.cpp:80-104).
int ref_mip(const double* vol, const int* dims, int axis, double* out) {
  return guarded([&] {
    VoxelGrid g({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    std::memcpy(g.data().data(), vol, g.data().size() * sizeof(double));
    VoxelGrid r = post::mip(g, axis);
    std::memcpy(out, r.data().data(), r.data().size() * sizeof(double));
  });
}

// ground_truth_pd (render.cpp:106-145): xyz [sum(counts)][3] blood scatterer
// positions, counts[f] of them in frame f.
int ref_ground_truth_pd(const double* xyz, const int* counts, int n_frames, const int* dims,
                        const double* spacing, const double* origin, double sigma_voxels,
                        double* out) {
  return guarded([&] {
    std::vector<std::vector<Vec3>> frames(static_cast<std::size_t>(n_frames));
    std::size_t k = 0;
    for (int f = 0; f < n_frames; ++f)
      for (int i = 0; i < counts[f]; ++i, ++k)
        frames[f].push_back(Vec3{xyz[3 * k], xyz[3 * k + 1], xyz[3 * k + 2]});
    beamform::GridSpec g;
    g.dims = {dims[0], dims[1], dims[2]};
    g.spacing = Vec3{spacing[0], spacing[1], spacing[2]};
    g.origin = Vec3{origin[0], origin[1], origin[2]};
    VoxelGrid r = post::ground_truth_pd(frames, g, sigma_voxels);
    std::memcpy(out, r.data().data(), r.data().size() * sizeof(double));
  });
}

// Writers, for byte-compatibility tests of the stage outputs
// (grid.cpp:79-99, render.cpp:147-175, das.cpp:395-407, metrics.cpp:114-126).
int ref_write_grid(const char* path, const int* dims, const double* sp, const double* org,
                   const double* data) {
  return guarded([&] {
    VoxelGrid g({dims[0], dims[1], dims[2]}, {sp[0], sp[1], sp[2]}, {org[0], org[1], org[2]});
    std::memcpy(g.data().data(), data, g.data().size() * sizeof(double));
    write_grid(path, g);
  });
}

int ref_write_pgm(const char* path, const int* dims, const double* data) {
  return guarded([&] {
    VoxelGrid g({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    std::memcpy(g.data().data(), data, g.data().size() * sizeof(double));
    post::write_pgm(path, g);
  });
}

int ref_write_iq_volume(const char* path, const int* dims, const double* sp, const double* org,
                        int frame_index, int n_angles, const double* iq) {
  return guarded([&] {
    beamform::IqVolume v;
    v.grid.dims = {dims[0], dims[1], dims[2]};
    v.grid.spacing = Vec3{sp[0], sp[1], sp[2]};
    v.grid.origin = Vec3{org[0], org[1], org[2]};
    v.frame_index = frame_index;
    v.n_angles = n_angles;
    const auto* src = reinterpret_cast<const std::complex<double>*>(iq);
    v.values.assign(src, src + v.grid.num_points());
    beamform::write_iq_volume(path, v);
  });
}

int ref_metrics_text(const double* test, const double* refimg, const int* dims, char* csv,
                     int csv_cap, char* js, int js_cap) {
  return guarded([&] {
    VoxelGrid a({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    VoxelGrid b({dims[0], dims[1], dims[2]}, {1, 1, 1}, {0, 0, 0});
    std::memcpy(a.data().data(), test, a.data().size() * sizeof(double));
    std::memcpy(b.data().data(), refimg, b.data().size() * sizeof(double));
    post::MetricsReport m = post::metrics(a, b);
    std::snprintf(csv, csv_cap, "%s", post::metrics_csv(m).c_str());
    std::snprintf(js, js_cap, "%s", post::metrics_json(m).c_str());
  });
}

// rf::simulate_rf / simulate_rf_chunked (simulate.cpp, compiled with the FFTW
// stub): one transmit of a scatterer cloud -> out [T][E]; td_params = half
// width, pitch, centre frequency, fractional bandwidth, elevation height,
// focus, core weight, tail weight, aperture factor; medium = c, attenuation,
// min_fs_ratio.  chunked: 0 simulate_rf, 1 simulate_rf_chunked(budget).
// stats_out: blocks, frequencies, peak_tracked_bytes, pair_bin_products.
int ref_simulate_rf(const double* pos, const double* refl, std::size_t n, int E,
                    const double* xyz, int subelements, const double* td_params,
                    const double* tx_delays, const double* tx_apod, double tx_angle,
                    const double* medium, std::size_t budget, double fs, double duration,
                    int chunked, std::size_t chunk_budget, double* out, int* n_samples,
                    std::uint64_t* stats_out) {
  return guarded([&] {
    rf::Transducer td = make_sim_probe(E, xyz, subelements, td_params);
    rf::TxEvent tx;
    tx.angle = tx_angle;
    tx.delays.assign(tx_delays, tx_delays + E);
    tx.apodization.assign(tx_apod, tx_apod + E);
    rf::MediumParams m;
    m.c = medium[0];
    m.attenuation_db_cm_mhz = medium[1];
    m.min_fs_ratio = medium[2];
    m.scatterer_memory_budget = budget;
    rf::RfSimStats st;
    tissue::ScattererCloud cloud = make_cloud(pos, refl, n);
    rf::RfFrame fr = chunked ? rf::simulate_rf_chunked(cloud, td, tx, m, fs, duration, chunk_budget, &st)
                             : rf::simulate_rf(cloud, td, tx, m, fs, duration, &st);
    *n_samples = fr.n_samples;
    if (out) std::memcpy(out, fr.samples.data(), fr.samples.size() * sizeof(double));
    if (stats_out) {
      stats_out[0] = st.blocks;
      stats_out[1] = st.frequencies;
      stats_out[2] = st.peak_tracked_bytes;
      stats_out[3] = st.pair_bin_products;
    }
  });
}

// rf::compose_frames (simulate.cpp): F frames; tissue / flow clouds given as
// concatenated positions [sum counts][3] and reflectivities with per-frame
// counts.  out [F][T][E]; stats_out: tissue_simulations, flow_simulations.
int ref_compose_frames(const double* t_pos, const double* t_refl, const int* t_counts,
                       const double* f_pos, const double* f_refl, const int* f_counts, int F,
                       int static_tissue, int E, const double* xyz, int subelements,
                       const double* td_params, const double* tx_delays, const double* tx_apod,
                       double tx_angle, const double* medium, std::size_t budget, double fs,
                       double duration, double* out, int* n_samples, int* stats_out) {
  return guarded([&] {
    rf::Transducer td = make_sim_probe(E, xyz, subelements, td_params);
    rf::TxEvent tx;
    tx.angle = tx_angle;
    tx.delays.assign(tx_delays, tx_delays + E);
    tx.apodization.assign(tx_apod, tx_apod + E);
    rf::MediumParams m;
    m.c = medium[0];
    m.attenuation_db_cm_mhz = medium[1];
    m.min_fs_ratio = medium[2];
    m.scatterer_memory_budget = budget;
    std::vector<tissue::ScattererCloud> tf, ff;
    std::size_t ot = 0, of = 0;
    for (int f = 0; f < F; ++f) {
      tf.push_back(make_cloud(t_pos + 3 * ot, t_refl + ot, t_counts[f]));
      ff.push_back(make_cloud(f_pos + 3 * of, f_refl + of, f_counts[f]));
      ot += t_counts[f];
      of += f_counts[f];
    }
    rf::ComposeStats st;
    std::vector<rf::RfFrame> fr =
        rf::compose_frames(tf, ff, static_tissue != 0, td, tx, m, fs, duration, &st);
    *n_samples = fr.empty() ? 0 : fr[0].n_samples;
    if (out)
      for (int f = 0; f < F; ++f)
        std::memcpy(out + (std::size_t)f * fr[f].samples.size(), fr[f].samples.data(),
                    fr[f].samples.size() * sizeof(double));
    stats_out[0] = st.tissue_simulations;
    stats_out[1] = st.flow_simulations;
  });
}

// build_delay_matrix (das.cpp:126-208) over voxels [n][3] for one transmit:
// the CSR is kept per thread; ref_delay_matrix_build returns nnz (or -1) and
// ref_delay_matrix_fetch copies row_ptr [n + 1], col_idx [nnz], values
// [nnz][2], out_of_window and padded_samples.
thread_local beamform::DelayMatrix g_dm;

long long ref_delay_matrix_build(const double* voxels, std::size_t n, double angle, double t0,
                                 double fs, int T, int E, const double* elements, double c,
                                 double fc, double f_number, int interp) {
  const int rc = guarded([&] {
    rf::Transducer td = make_probe(E, elements, fc);
    std::vector<Vec3> vox(n);
    for (std::size_t i = 0; i < n; ++i) vox[i] = {voxels[3 * i], voxels[3 * i + 1], voxels[3 * i + 2]};
    rf::TxEvent tx;
    tx.angle = angle;
    beamform::BeamformParams bp;
    bp.c = c;
    bp.center_frequency = fc;
    bp.f_number = f_number;
    bp.interp_order = interp;
    g_dm = beamform::build_delay_matrix(vox, tx, td, bp, fs, t0, T);
  });
  return rc ? -1 : static_cast<long long>(g_dm.col_idx.size());
}

void ref_delay_matrix_fetch(std::uint64_t* row_ptr, std::int32_t* col_idx, double* values,
                            std::uint64_t* out_of_window, int* padded_samples) {
  for (std::size_t i = 0; i < g_dm.row_ptr.size(); ++i) row_ptr[i] = g_dm.row_ptr[i];
  std::memcpy(col_idx, g_dm.col_idx.data(), g_dm.col_idx.size() * sizeof(std::int32_t));
  std::memcpy(values, g_dm.values.data(), g_dm.values.size() * sizeof(std::complex<double>));
  *out_of_window = g_dm.out_of_window;
  *padded_samples = g_dm.padded_samples;
}

}  // extern "C"
