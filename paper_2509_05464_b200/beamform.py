"""fqf::beamform on the B200: the reference's beamforming API
(proj/include/fqf/beamform/{iq,das}.hpp) over the C ABI in include/fqfgpu.h.

Same names, argument meaning and error behaviour as the reference:

  rf_to_iq(rf, f_c, lowpass_taps=33) -> IqFrame              iq.hpp:31 / iq.cpp:34-82
  plan_chunks(n_points, n_angles, budget_bytes) -> ChunkPlan  das.hpp:49 / das.cpp:97-119
  das_reconstruct(frames, grid, td, bp, opts, stats) -> [IqVolume]
                                                              das.hpp:124-127 / das.cpp:224-356
  assemble_frames(work_dir, plan, grid, n_frames)             das.hpp:131-132 / das.cpp:358-393
  write_iq_volume / read_iq_volume                            das.hpp:134-135 / das.cpp:395-429

Contract violations raise ``Error`` (fqf::Error) with the reference's
require() message.  All arithmetic runs in the CUDA library; this module only
validates, marshals and does the reference's file I/O.  IQ values come back
as complex128 like IqVolume::values (converted from the GPU's complex64).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import tempfile
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import fqf1
from ._native import (Bf, DasOpts, DasStats as _CStats, Error, Grid, Probe, RfDesc, check, load)

__all__ = ["Error", "GridSpec", "Transducer", "TxEvent", "RfFrame", "IqFrame", "BeamformParams",
           "DasOptions", "DasStats", "IqVolume", "ChunkPlan", "rf_to_iq", "plan_chunks",
           "das_reconstruct", "das_reconstruct_array", "assemble_frames", "write_iq_volume",
           "read_iq_volume", "plane_wave_delays", "matrix32x32", "l11_4v", "validate_transducer"]


def _require(cond, msg):
    if not cond:
        raise Error(msg)


@dataclass
class GridSpec:
    """Reconstruction grid (das.hpp:20-33); voxel index i + nx*(j + ny*k)."""
    dims: Tuple[int, int, int] = (0, 0, 0)
    spacing: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)

    def num_points(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def point(self, flat: int):
        nx, ny = self.dims[0], self.dims[1]
        i, j, k = flat % nx, (flat // nx) % ny, flat // (nx * ny)
        return (self.origin[0] + i * self.spacing[0], self.origin[1] + j * self.spacing[1],
                self.origin[2] + k * self.spacing[2])

    def _c(self) -> Grid:
        return Grid((C.c_int * 3)(*map(int, self.dims)), (C.c_double * 3)(*self.spacing),
                    (C.c_double * 3)(*self.origin))


@dataclass
class Transducer:
    """Probe geometry (rf/transducer.hpp:13-31).  DAS reads the element
    centres only (das.cpp:137-145); the RF simulator (rf.py) reads all."""
    elements: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    name: str = ""
    pitch: float = 0.3e-3
    center_frequency: float = 0.0
    half_width: float = 0.0
    subelements: int = 4
    fractional_bandwidth: float = 0.67
    elevation_height: float = 0.0
    elevation_focus: float = 0.0
    elevation_core_weight: float = 0.85
    elevation_tail_weight: float = 0.15
    elevation_aperture_factor: float = 0.494

    def n_elements(self) -> int:
        return int(np.asarray(self.elements).shape[0])


def validate_transducer(t: Transducer) -> None:
    """transducer.cpp:10-24 (same messages)."""
    _require(t.n_elements() > 0, "transducer has no elements")
    _require(t.half_width > 0.0, "element half-width must be positive")
    _require(t.subelements >= 1, "sub-element count must be at least 1")
    _require(t.pitch > 0.0, "pitch must be positive")
    _require(t.center_frequency > 0.0, "center frequency must be positive")
    _require(0.0 < t.fractional_bandwidth < 2.0, "fractional bandwidth must lie in (0, 2)")
    if t.elevation_height > 0.0:
        _require(t.elevation_focus > 0.0, "elevation focus must be positive when a lens is present")
        _require(t.elevation_aperture_factor > 0.0, "elevation aperture factor must be positive")
        _require(t.elevation_core_weight >= 0.0 and t.elevation_tail_weight >= 0.0,
                 "elevation weights must be nonnegative")


def matrix32x32() -> Transducer:
    """32 x 32 matrix preset (transducer.cpp:43-60): j outer, i inner."""
    el = np.array([[(i - 15.5) * 0.3e-3, (j - 15.5) * 0.3e-3, 0.0]
                   for j in range(32) for i in range(32)])
    return Transducer(el, "matrix32x32", 0.3e-3, 3.0e6, half_width=0.135e-3, subelements=2,
                      fractional_bandwidth=0.6)


def l11_4v() -> Transducer:
    """128-element linear preset (transducer.cpp:26-41)."""
    el = np.array([[(n - 63.5) * 0.3e-3, 0.0, 0.0] for n in range(128)])
    return Transducer(el, "l11-4v", 0.3e-3, 7.7e6, half_width=0.135e-3, subelements=4,
                      fractional_bandwidth=0.67, elevation_height=5.0e-3, elevation_focus=18.0e-3)


@dataclass
class TxEvent:
    """One steered plane-wave transmit (transducer.hpp:42-46)."""
    angle: float = 0.0
    delays: Optional[np.ndarray] = None
    apodization: Optional[np.ndarray] = None


def plane_wave_delays(td: Transducer, angle: float, c: float) -> TxEvent:
    """transducer.cpp:62-78."""
    validate_transducer(td)
    _require(c > 0.0, "sound speed must be positive")
    _require(abs(angle) < 1.5707963267948966, "steering angle must lie in (-pi/2, pi/2)")
    d = np.asarray(td.elements)[:, 0] * (math.sin(angle) / c)
    return TxEvent(angle, d - d.min(), np.ones(len(d)))


@dataclass
class RfFrame:
    """One received frame, time-major samples [T][E] (simulate.hpp:22-37)."""
    samples: np.ndarray
    sampling_rate: float
    t0: float = 0.0
    tx: TxEvent = field(default_factory=TxEvent)

    @property
    def n_samples(self) -> int:
        return int(self.samples.shape[0])

    @property
    def n_elements(self) -> int:
        return int(self.samples.shape[1]) if self.samples.ndim == 2 else 0


@dataclass
class IqFrame:
    """Complex baseband frame [T][E] (iq.hpp:13-24)."""
    samples: np.ndarray
    sampling_rate: float
    t0: float
    center_frequency: float

    @property
    def n_samples(self):
        return int(self.samples.shape[0])

    @property
    def n_elements(self):
        return int(self.samples.shape[1])

    def at(self, t, e):
        return self.samples[t, e]


@dataclass
class BeamformParams:
    """das.hpp:76-82."""
    c: float = 1540.0
    center_frequency: float = 0.0
    f_number: float = 1.5
    interp_order: int = 1
    lowpass_taps: int = 33

    def _c(self) -> Bf:
        return Bf(self.c, self.center_frequency, self.f_number, int(self.interp_order),
                  int(self.lowpass_taps))


@dataclass
class DasOptions:
    """das.hpp:101-108."""
    memory_budget_bytes: int = 100_000_000
    matrix_budget_bytes: int = 512_000_000
    cache_matrices: bool = True
    work_dir: str = ""
    write_frames: bool = False
    keep_chunk_files: bool = False


@dataclass
class DasStats:
    """das.hpp:110-116."""
    chunks: int = 0
    matrix_builds: int = 0
    out_of_window: int = 0
    matrix_bytes_peak: int = 0
    accumulator_bytes_peak: int = 0


@dataclass
class IqVolume:
    """das.hpp:94-99."""
    grid: GridSpec
    frame_index: int = 0
    n_angles: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))


@dataclass
class ChunkPlan:
    """das.hpp:39-47."""
    n_points: int = 0
    n_angles: int = 0
    budget_bytes: int = 0
    n_chunks: int = 0
    ranges: List[Tuple[int, int]] = field(default_factory=list)

    def max_chunk_points(self) -> int:
        return max((e - b for b, e in self.ranges), default=0)


# ------------------------------------------------------------------ demod --

def rf_to_iq(rf: RfFrame, f_c: float, lowpass_taps: int = 33) -> IqFrame:
    """iq.cpp:34-82 on the GPU (complex64 precision, returned as complex128)."""
    return rf_to_iq_batch([rf], f_c, lowpass_taps)[0]


def rf_to_iq_batch(frames: Sequence[RfFrame], f_c: float, lowpass_taps: int = 33):
    frames = list(frames)
    _require(len(frames) > 0, "frame has no samples")
    T, E = frames[0].samples.shape if frames[0].samples.ndim == 2 else (0, 0)
    fs = frames[0].sampling_rate
    for fr in frames:
        _require(fr.samples.ndim == 2 and fr.samples.shape == (T, E), "frame has no samples")
        _require(fr.sampling_rate == fs, "sampling rate differs between frames")
    rf = np.ascontiguousarray(np.stack([fr.samples for fr in frames]), dtype=np.float32)
    t0 = np.ascontiguousarray([fr.t0 for fr in frames], dtype=np.float64)
    out = np.empty(rf.shape + (2,), dtype=np.float32)
    L = load()
    if T == 0 or E == 0:
        raise Error("frame has no samples")
    check(L.fqfg_rf_to_iq(rf.ctypes.data, len(frames), T, E, fs, t0.ctypes.data, f_c,
                          lowpass_taps, out.ctypes.data))
    iq = out[..., 0].astype(np.float64) + 1j * out[..., 1].astype(np.float64)
    return [IqFrame(iq[b], fs, frames[b].t0, f_c) for b in range(len(frames))]


# ------------------------------------------------------------------- plan --

def plan_chunks(n_points: int, n_angles: int, budget_bytes: int) -> ChunkPlan:
    L = load()
    k = C.c_size_t(0)
    check(L.fqfg_plan_chunks(n_points, n_angles, budget_bytes, None, 0, C.byref(k)))
    r = np.zeros(2 * k.value, dtype=np.uint64)
    check(L.fqfg_plan_chunks(n_points, n_angles, budget_bytes, r.ctypes.data, k.value,
                             C.byref(k)))
    return ChunkPlan(n_points, n_angles, budget_bytes, int(k.value),
                     [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(k.value)])


# -------------------------------------------------------------------- DAS --

def _desc(F, A, T, E, fs, t0, angles):
    t0 = np.ascontiguousarray(np.broadcast_to(np.asarray(t0, np.float64), (A,)))
    angles = np.ascontiguousarray(angles, dtype=np.float64)
    d = RfDesc(F, A, T, E, fs, t0.ctypes.data_as(C.POINTER(C.c_double)),
               angles.ctypes.data_as(C.POINTER(C.c_double)))
    return d, (t0, angles)


def _probe(elements):
    el = np.ascontiguousarray(elements, dtype=np.float64).reshape(-1, 3)
    return Probe(el.shape[0], el.ctypes.data_as(C.POINTER(C.c_double))), el


def das_reconstruct_array(rf: np.ndarray, sampling_rate: float, t0, angles, grid: GridSpec,
                          elements, bp: BeamformParams, opts: Optional[DasOptions] = None,
                          want_stats: bool = False):
    """Array form of das_reconstruct: rf [F][A][T][E] (f32) -> (iq [F][N]
    complex64, DasStats | None).  The host-side file options are ignored."""
    opts = opts or DasOptions()
    rf = np.ascontiguousarray(rf, dtype=np.float32)
    _require(rf.ndim == 4, "rf must be [frames][angles][samples][elements]")
    F, A, T, E = rf.shape
    desc, keep = _desc(F, A, T, E, sampling_rate, t0, angles)
    probe, el = _probe(elements)
    g = grid._c()
    b = bp._c()
    o = DasOpts(int(opts.memory_budget_bytes), int(opts.matrix_budget_bytes),
                int(bool(opts.cache_matrices)))
    N = grid.num_points()
    out = np.empty((F, max(N, 0), 2), dtype=np.float32)
    st = _CStats()
    check(load().fqfg_das(C.byref(desc), rf.ctypes.data, C.byref(g), C.byref(probe), C.byref(b),
                          C.byref(o), out.ctypes.data, C.byref(st) if want_stats else None))
    iq = out.view(np.complex64).reshape(F, N)
    stats = None
    if want_stats:
        stats = DasStats(int(st.chunks), int(st.matrix_builds), int(st.out_of_window),
                         int(st.matrix_bytes_peak), int(st.accumulator_bytes_peak))
    return iq, stats


def das_reconstruct(frames: Sequence[Sequence[RfFrame]], grid: GridSpec, td: Transducer,
                    bp: BeamformParams, opts: Optional[DasOptions] = None,
                    stats: Optional[DasStats] = None) -> List[IqVolume]:
    """das.cpp:224-356: frames[frame][angle] -> one IqVolume per frame."""
    opts = opts or DasOptions()
    _require(len(frames) > 0, "no frames to reconstruct")
    F, A = len(frames), len(frames[0])
    _require(A >= 1, "frames carry no transmits")
    E = td.n_elements()
    _require(E >= 1, "transducer has no elements")
    first = frames[0][0]
    fs, T = first.sampling_rate, first.n_samples
    _require(fs > 0.0 and T >= 1, "frames are empty")
    for f in range(F):
        _require(len(frames[f]) == A, "transmit count differs between frames")
        for a in range(A):
            fr = frames[f][a]
            _require(fr.sampling_rate == fs, "sampling rate differs between frames")
            _require(fr.n_samples == T, "sample count differs between frames")
            _require(fr.n_elements == E, "element count does not match the transducer")
            _require(fr.tx.angle == frames[0][a].tx.angle,
                     "transmit angle differs between frames at the same slot")
            _require(fr.t0 == frames[0][a].t0,
                     "start time differs between frames at the same slot")
    rf = np.empty((F, A, T, E), dtype=np.float32)
    for f in range(F):
        for a in range(A):
            rf[f, a] = frames[f][a].samples
    angles = [frames[0][a].tx.angle for a in range(A)]
    t0 = [frames[0][a].t0 for a in range(A)]
    iq, st = das_reconstruct_array(rf, fs, t0, angles, grid, td.elements, bp, opts,
                                   want_stats=True)
    vols = [IqVolume(grid, f, A, iq[f].astype(np.complex128)) for f in range(F)]
    _persist(vols, grid, A, opts, st)
    if stats is not None:
        stats.__dict__.update(st.__dict__)
    return vols


def _persist(vols, grid, A, opts, st):
    """Honour DasOptions' file side effects (das.cpp:280-352): chunk stripes
    IQ_CHUNK_k.fqf when keep_chunk_files, Frame_i.fqf when write_frames."""
    if not (opts.write_frames or opts.keep_chunk_files):
        return
    d = opts.work_dir or tempfile.mkdtemp(prefix="fqf_das_")
    os.makedirs(d, exist_ok=True)
    if opts.keep_chunk_files:
        plan = plan_chunks(grid.num_points(), A, opts.memory_budget_bytes)
        # das.cpp may re-plan for the matrix budget; st.chunks is authoritative.
        if st is not None and st.chunks != plan.n_chunks:
            plan = ChunkPlan(plan.n_points, A, plan.budget_bytes, st.chunks,
                             _split_ranges(plan.n_points, st.chunks))
        F = len(vols)
        for ci, (b, e) in enumerate(plan.ranges):
            stripe = np.concatenate([v.values[b:e] for v in vols])
            fqf1.write_container(os.path.join(d, f"IQ_CHUNK_{ci + 1}.fqf"),
                                 [("kind", "iq_chunk"), ("chunk", str(ci + 1)),
                                  ("begin", str(b)), ("end", str(e)), ("frames", str(F)),
                                  ("n_angles", str(A))], stripe.astype(np.complex128))
    if opts.write_frames:
        for f, v in enumerate(vols):
            write_iq_volume(os.path.join(d, f"Frame_{f + 1}.fqf"), v)


def _split_ranges(n, k):
    base, rem, at, out = n // k, n % k, 0, []
    for i in range(k):
        ln = base + (1 if i < rem else 0)
        out.append((at, at + ln))
        at += ln
    return out


def assemble_frames(work_dir: str, plan: ChunkPlan, grid: GridSpec, n_frames: int):
    """das.cpp:358-393."""
    _require(n_frames >= 1, "no frames to assemble")
    _require(plan.n_points == grid.num_points(), "chunk plan does not match the grid")
    _require(plan.n_chunks == len(plan.ranges), "chunk plan is inconsistent")
    vols = [IqVolume(grid, f, 0, np.zeros(plan.n_points, np.complex128)) for f in range(n_frames)]
    for ci, (b, e) in enumerate(plan.ranges):
        path = os.path.join(work_dir, f"IQ_CHUNK_{ci + 1}.fqf")
        _require(os.path.exists(path), f"missing chunk file {path}")
        h, payload = fqf1.read_container(path)
        hv = lambda k: fqf1.header_value(h, k)  # noqa: E731
        _require(hv("kind") == "iq_chunk", f"{path}: not a chunk file")
        _require(int(hv("chunk")) == ci + 1, f"{path}: chunk index mismatch")
        _require(int(hv("begin")) == b and int(hv("end")) == e,
                 f"{path}: chunk range does not match the plan")
        _require(int(hv("frames")) == n_frames, f"{path}: frame count mismatch")
        na = int(hv("n_angles"))
        data = fqf1.as_complex128(payload)
        _require(data.size == (e - b) * n_frames, f"{path}: payload does not match the chunk shape")
        for f in range(n_frames):
            vols[f].n_angles = na
            vols[f].values[b:e] = data[f * (e - b):(f + 1) * (e - b)]
    return vols


def write_iq_volume(path: str, vol: IqVolume) -> None:
    """das.cpp:395-407."""
    _require(vol.values.size == vol.grid.num_points(), "volume values do not match the grid dims")
    g = vol.grid
    fqf1.write_container(path, [
        ("kind", "iq_volume"), ("dims", f"{g.dims[0]} {g.dims[1]} {g.dims[2]}"),
        ("spacing", " ".join(fqf1.fmt17(v) for v in g.spacing)),
        ("origin", " ".join(fqf1.fmt17(v) for v in g.origin)),
        ("frame", str(vol.frame_index + 1)), ("n_angles", str(vol.n_angles))],
        np.asarray(vol.values, dtype=np.complex128))


def read_iq_volume(path: str) -> IqVolume:
    """das.cpp:409-429."""
    h, payload = fqf1.read_container(path)
    hv = lambda k: fqf1.header_value(h, k)  # noqa: E731
    _require(hv("kind") == "iq_volume", f"{path}: not a volume container")
    dims = tuple(int(x) for x in hv("dims").split())
    g = GridSpec(dims, tuple(float(x) for x in hv("spacing").split()),
                 tuple(float(x) for x in hv("origin").split()))
    v = IqVolume(g, int(hv("frame")) - 1, int(hv("n_angles")), fqf1.as_complex128(payload))
    _require(v.values.size == g.num_points(), f"{path}: payload does not match the grid dims")
    return v
