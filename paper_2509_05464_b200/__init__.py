"""B200-native (sm_100a) reconstruction hot path of 3D-FQFlow (arXiv 2509.05464).

RF channel data -> IQ demodulation -> 3D plane-wave delay-and-sum with angle
compounding -> Casorati SVD clutter filter -> power Doppler, behind the
reference's own API (fqf::beamform / fqf::post), implemented as hand-written
CUDA kernels in libfqfgpu.so (C ABI: include/fqfgpu.h).
"""
from ._native import Error, device_count  # noqa: F401
from .beamform import (BeamformParams, ChunkPlan, DasOptions, DasStats, GridSpec,  # noqa: F401
                       IqFrame, IqVolume, RfFrame, Transducer, TxEvent, assemble_frames,
                       das_reconstruct, das_reconstruct_array, l11_4v, matrix32x32, plan_chunks,
                       plane_wave_delays, read_iq_volume, rf_to_iq, write_iq_volume)
from .post import SvdReport, power_doppler, svd_filter  # noqa: F401
