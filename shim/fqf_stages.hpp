// fqf_stages.hpp -- the reference pipeline's beamform + post stage bodies
// (proj/src/pipeline/run.cpp:397-487) fused on the GPU: the declarations a
// maintainer calls from run_beamform / run_post.
#pragma once

#include <string>
#include <vector>

#include "fqf/beamform/das.hpp"
#include "fqf/rf/transducer.hpp"

namespace fqf::gpu {

// The RunConfig fields run_beamform / run_post read (run.cpp:397-487).
struct StageConfig {
  rf::Transducer transducer;
  beamform::GridSpec grid;
  int n_frames = 0;
  std::vector<double> angles_deg;
  double sound_speed = 1540.0;
  double f_number = 1.5;
  int lowpass_taps = 33;
  double bmode_dynamic_range_db = 60.0;
  double pd_dynamic_range_db = 60.0;
  int svd_lo = 2;
  int svd_hi = 0;  // 0 = n_frames (run.cpp:457)
  double ground_truth_sigma_voxels = 1.0;
};

// rf/frame_FFFF_tx_AA.fqf + particles/frame_FFFF.fqf under `out` ->
// beamform/Frame_<f+1>.fqf (when write_frames), post/{bmode,pd,gt}.{fqf,pgm}
// and post/svd_report.json, the reference's files.  One reconstruction
// engine pass: the IQ ensemble stays on the GPU between beamforming and the
// clutter filter (no F-volume round trip through the file system or the
// host, run.cpp:438-440).  Returns the written paths relative to `out`.
std::vector<std::string> run_beamform_post(const std::string& out, const StageConfig& cfg,
                                           bool write_frames = true);

}  // namespace fqf::gpu
