"""ctypes binding of the C ABI in include/fqfgpu.h (libfqfgpu.so, sm_100a).

The library is built in-tree by ``paper_2509_05464_b200/csrc/Makefile`` (see
``__graft_entry__.build``).  There is no CPU implementation behind any of
these symbols: on a machine without an sm_100 device every compute entry
point fails with FQFG_ENODEV and the Python layer raises ``Error``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfqfgpu.so")

FQFG_OK, FQFG_EINVAL, FQFG_ECUDA, FQFG_ENODEV, FQFG_ENOMEM = range(5)

# Every symbol include/fqfgpu.h declares (tests/test_capi.py checks the
# header and this list agree and that the built library exports them all).
EXPORTS = (
    "fqfg_last_error", "fqfg_version", "fqfg_device_count", "fqfg_set_device",
    "fqfg_rf_to_iq", "fqfg_plan_chunks", "fqfg_das", "fqfg_svd_filter", "fqfg_power_doppler",
    "fqfg_reconstruct_pd", "fqfg_das_plan_create", "fqfg_das_plan_info_get",
    "fqfg_das_plan_destroy", "fqfg_das_dev", "fqfg_gram_work_bytes", "fqfg_gram_dev",
    "fqfg_eig_dev", "fqfg_eig_band_dev", "fqfg_project_pd_dev", "fqfg_synth_rf_dev", "fqfg_das_plan_set_timing",
    "fqfg_das_last_timing", "fqfg_launch_count", "fqfg_build_delay_matrix",
    "fqfg_apply_delay_matrix", "fqfg_das_slab_samples", "fqfg_copy_slices_h2d",
    "fqfg_render_db", "fqfg_render_db_dev", "fqfg_bmode", "fqfg_mip", "fqfg_ground_truth_pd",
    "fqfg_metrics", "fqfg_metrics_dev", "fqfg_plan_rf_chunks", "fqfg_simulate_rf",
    "fqfg_simulate_rf_dev", "fqfg_nccl_unique_id", "fqfg_recon_create", "fqfg_recon_info_get",
    "fqfg_recon_run", "fqfg_recon_run_dev", "fqfg_recon_set_timing", "fqfg_recon_last_timing",
    "fqfg_recon_mma_blocks",
    "fqfg_recon_destroy", "fqfg_recon_copy_iq", "fqfg_recon_report", "fqfg_gram_tc_work_bytes", "fqfg_gram_tc_dev",
)


class Error(RuntimeError):
    """A failed call (the Python face of fqf::Error / a nonzero status)."""

    def __init__(self, msg, code=FQFG_EINVAL):
        super().__init__(msg)
        self.code = code


class Grid(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("spacing", C.c_double * 3), ("origin", C.c_double * 3)]


class Probe(C.Structure):
    _fields_ = [("n_elements", C.c_int), ("xyz", C.POINTER(C.c_double))]


class Bf(C.Structure):
    _fields_ = [("c", C.c_double), ("center_frequency", C.c_double), ("f_number", C.c_double),
                ("interp_order", C.c_int), ("lowpass_taps", C.c_int)]


class RfDesc(C.Structure):
    _fields_ = [("n_frames", C.c_int), ("n_angles", C.c_int), ("n_samples", C.c_int),
                ("n_elements", C.c_int), ("sampling_rate", C.c_double),
                ("t0", C.POINTER(C.c_double)), ("angles", C.POINTER(C.c_double))]


class DasOpts(C.Structure):
    _fields_ = [("memory_budget_bytes", C.c_size_t), ("matrix_budget_bytes", C.c_size_t),
                ("cache_matrices", C.c_int)]


class DasStats(C.Structure):
    _fields_ = [("chunks", C.c_uint64), ("matrix_builds", C.c_uint64),
                ("out_of_window", C.c_uint64), ("matrix_bytes_peak", C.c_uint64),
                ("accumulator_bytes_peak", C.c_uint64)]


class TransducerC(C.Structure):
    _fields_ = [("n_elements", C.c_int), ("xyz", C.POINTER(C.c_double)),
                ("half_width", C.c_double), ("subelements", C.c_int), ("pitch", C.c_double),
                ("center_frequency", C.c_double), ("fractional_bandwidth", C.c_double),
                ("elevation_height", C.c_double), ("elevation_focus", C.c_double),
                ("elevation_core_weight", C.c_double), ("elevation_tail_weight", C.c_double),
                ("elevation_aperture_factor", C.c_double)]


class MediumC(C.Structure):
    _fields_ = [("c", C.c_double), ("attenuation_db_cm_mhz", C.c_double),
                ("scatterer_memory_budget", C.c_size_t), ("min_fs_ratio", C.c_double)]


class RfSimStatsC(C.Structure):
    _fields_ = [("blocks", C.c_int), ("frequencies", C.c_int),
                ("peak_tracked_bytes", C.c_size_t), ("pair_bin_products", C.c_uint64)]


class RfChunkPlanC(C.Structure):
    _fields_ = [("blocks", C.c_int), ("block_scatterers", C.c_size_t),
                ("per_scatterer_bytes", C.c_size_t), ("fixed_bytes", C.c_size_t)]


class PlanInfo(C.Structure):
    _fields_ = [("n_points", C.c_size_t), ("frames_per_pass", C.c_int), ("n_passes", C.c_int),
                ("work_bytes", C.c_size_t), ("active_pairs", C.c_uint64), ("tile", C.c_int * 3),
                ("shape", C.c_int * 4), ("mode", C.c_int)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class ReconOpts(C.Structure):
    _fields_ = [("keep_lo", C.c_int), ("keep_hi", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_id", C.c_void_p), ("allreduce", ALLREDUCE_FN),
                ("allreduce_user", C.c_void_p), ("device_budget", C.c_size_t),
                ("ring_frames", C.c_int), ("x_buffers", C.c_int), ("gram_fp64", C.c_int),
                ("rf_broadcast", C.c_int)]


class ReconInfo(C.Structure):
    _fields_ = [("k_begin", C.c_int), ("k_end", C.c_int), ("v_begin", C.c_size_t),
                ("v_end", C.c_size_t), ("t_begin", C.c_int), ("t_end", C.c_int),
                ("frames_per_pass", C.c_int), ("n_passes", C.c_int), ("x_buffers", C.c_int),
                ("ring_frames", C.c_int), ("device_bytes", C.c_size_t),
                ("h2d_bytes_per_ensemble", C.c_size_t), ("active_samples", C.c_uint64),
                ("tile", C.c_int * 3), ("shape", C.c_int * 4), ("nccl", C.c_int),
                ("gram_fp64", C.c_int), ("mode", C.c_int)]


_lib = None


def load() -> C.CDLL:
    """Load libfqfgpu.so (raises Error if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise Error(f"{LIB_PATH} is not built; run __graft_entry__.build()", FQFG_ENODEV)
    L = C.CDLL(LIB_PATH)
    vp, sz, i, d = C.c_void_p, C.c_size_t, C.c_int, C.c_double
    L.fqfg_last_error.restype = C.c_char_p
    L.fqfg_rf_to_iq.argtypes = [vp, i, i, i, d, vp, d, i, vp]
    L.fqfg_plan_chunks.argtypes = [sz, i, sz, vp, sz, C.POINTER(sz)]
    L.fqfg_das.argtypes = [C.POINTER(RfDesc), vp, C.POINTER(Grid), C.POINTER(Probe), C.POINTER(Bf),
                           C.POINTER(DasOpts), vp, C.POINTER(DasStats)]
    L.fqfg_svd_filter.argtypes = [vp, i, sz, i, i, vp, vp, vp, vp]
    L.fqfg_build_delay_matrix.argtypes = [vp, sz, d, d, d, i, C.POINTER(Probe), C.POINTER(Bf),
                                          vp, vp, vp, vp, vp]
    L.fqfg_apply_delay_matrix.argtypes = [sz, vp, vp, vp, vp, sz, vp]
    L.fqfg_power_doppler.argtypes = [vp, i, sz, vp]
    L.fqfg_reconstruct_pd.argtypes = [C.POINTER(RfDesc), vp, C.POINTER(Grid), C.POINTER(Probe),
                                      C.POINTER(Bf), i, i, vp, vp, vp]
    L.fqfg_das_plan_create.argtypes = [C.POINTER(RfDesc), C.POINTER(Grid), C.POINTER(Probe),
                                       C.POINTER(Bf), C.POINTER(vp)]
    L.fqfg_das_plan_info_get.argtypes = [vp, C.POINTER(PlanInfo)]
    L.fqfg_das_plan_destroy.argtypes = [vp]
    L.fqfg_das_plan_destroy.restype = None
    L.fqfg_das_dev.argtypes = [vp, vp, i, i, vp, vp, vp, vp]
    L.fqfg_gram_work_bytes.argtypes = [i]
    L.fqfg_gram_work_bytes.restype = sz
    L.fqfg_gram_dev.argtypes = [vp, i, sz, sz, sz, vp, vp, vp]
    L.fqfg_gram_tc_work_bytes.argtypes = [i]
    L.fqfg_gram_tc_work_bytes.restype = sz
    L.fqfg_gram_tc_dev.argtypes = [vp, i, sz, sz, sz, vp, vp, vp]
    L.fqfg_eig_dev.argtypes = [vp, i, vp, vp, vp]
    L.fqfg_eig_band_dev.argtypes = [vp, i, i, i, vp, vp, vp]
    L.fqfg_project_pd_dev.argtypes = [vp, i, sz, sz, sz, vp, i, i, vp, vp, vp]
    L.fqfg_synth_rf_dev.argtypes = [vp, sz, C.c_uint64, vp]
    L.fqfg_das_plan_set_timing.argtypes = [vp, i]
    L.fqfg_das_last_timing.argtypes = [vp, C.POINTER(d), C.POINTER(d)]
    L.fqfg_launch_count.restype = C.c_uint64
    L.fqfg_das_slab_samples.argtypes = [vp, i, i, C.POINTER(i), C.POINTER(i)]
    L.fqfg_copy_slices_h2d.argtypes = [vp, vp, sz, sz, sz, sz, vp]
    ip = C.POINTER(C.c_int)
    L.fqfg_render_db.argtypes = [vp, ip, d, i, vp]
    L.fqfg_render_db_dev.argtypes = [vp, sz, d, i, vp, vp]
    L.fqfg_bmode.argtypes = [vp, ip, d, vp]
    L.fqfg_mip.argtypes = [vp, ip, i, vp]
    L.fqfg_ground_truth_pd.argtypes = [vp, ip, i, C.POINTER(Grid), d, vp]
    L.fqfg_metrics.argtypes = [vp, vp, ip, vp]
    L.fqfg_metrics_dev.argtypes = [vp, vp, ip, vp, vp]
    L.fqfg_plan_rf_chunks.argtypes = [C.POINTER(TransducerC), sz, C.POINTER(MediumC), d, d, sz,
                                      C.POINTER(RfChunkPlanC)]
    L.fqfg_simulate_rf.argtypes = [vp, vp, sz, C.POINTER(TransducerC), vp, vp, C.POINTER(MediumC),
                                   d, d, i, sz, vp, C.POINTER(i), C.POINTER(RfSimStatsC)]
    L.fqfg_simulate_rf_dev.argtypes = [vp, vp, sz, C.POINTER(TransducerC), vp, vp, vp,
                                       C.POINTER(MediumC), d, d, vp, vp, vp]
    L.fqfg_nccl_unique_id.argtypes = [vp]
    L.fqfg_recon_create.argtypes = [C.POINTER(RfDesc), C.POINTER(Grid), C.POINTER(Probe),
                                    C.POINTER(Bf), C.POINTER(ReconOpts), C.POINTER(vp)]
    L.fqfg_recon_info_get.argtypes = [vp, C.POINTER(ReconInfo)]
    L.fqfg_recon_run.argtypes = [vp, i, vp, vp, vp]
    L.fqfg_recon_run_dev.argtypes = [vp, i, vp, vp]
    L.fqfg_recon_set_timing.argtypes = [vp, i]
    L.fqfg_recon_last_timing.argtypes = [vp, C.POINTER(d), C.POINTER(d), C.POINTER(d),
                                         C.POINTER(d)]
    L.fqfg_recon_mma_blocks.argtypes = [vp, C.POINTER(C.c_ulonglong)]
    L.fqfg_recon_copy_iq.argtypes = [vp, sz, sz, vp]
    L.fqfg_recon_report.argtypes = [vp, vp, vp]
    L.fqfg_recon_destroy.argtypes = [vp]
    L.fqfg_recon_destroy.restype = None
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != FQFG_OK:
        raise Error(load().fqfg_last_error().decode(), rc)


def device_count() -> int:
    try:
        return load().fqfg_device_count()
    except Error:
        return 0
