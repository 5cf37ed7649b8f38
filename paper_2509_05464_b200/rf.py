"""fqf::rf on the B200: the frequency-domain RF channel-data simulator
(rf/simulate.hpp, simulate.cpp) over the C ABI (csrc/rfsim.cu).

simulate_rf(cloud, transducer, tx, medium, fs, duration) -> RfFrame with
samples [T][E] (float64), T = round(fs * duration), t0 = 0, exactly the
reference's model: point scatterers, sub-element tiling, sinc directivity,
optional elevation lens, frequency-linear attenuation, Gaussian pulse,
inverse transform.  Same argument meaning and error messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._native import Error, MediumC, RfChunkPlanC, RfSimStatsC, TransducerC, check, load
from .beamform import RfFrame, Transducer, TxEvent, validate_transducer

__all__ = ["MediumParams", "ScattererCloud", "RfSimStats", "RfChunkPlan", "ComposeStats",
           "plan_rf_chunks", "simulate_rf", "simulate_rf_chunked", "compose_frames"]


@dataclass
class MediumParams:
    """simulate.hpp:15-20."""
    c: float = 1540.0
    attenuation_db_cm_mhz: float = 0.5
    scatterer_memory_budget: int = 2_000_000_000
    min_fs_ratio: float = 4.0

    def _c(self):
        return MediumC(self.c, self.attenuation_db_cm_mhz, int(self.scatterer_memory_budget),
                       self.min_fs_ratio)


@dataclass
class ScattererCloud:
    """tissue/cloud.hpp:14-20 (positions [n][3] m, reflectivity [n])."""
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    reflectivity: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(np.asarray(self.positions).reshape(-1, 3).shape[0])


@dataclass
class RfSimStats:
    """simulate.hpp:39-44."""
    blocks: int = 0
    frequencies: int = 0
    peak_tracked_bytes: int = 0
    pair_bin_products: int = 0


@dataclass
class RfChunkPlan:
    """simulate.hpp:63-68."""
    blocks: int = 0
    block_scatterers: int = 0
    per_scatterer_bytes: int = 0
    fixed_bytes: int = 0


@dataclass
class ComposeStats:
    """simulate.hpp:74-77."""
    tissue_simulations: int = 0
    flow_simulations: int = 0


def _td(t: Transducer):
    el = np.ascontiguousarray(np.asarray(t.elements, np.float64).reshape(-1, 3))
    return TransducerC(el.shape[0], el.ctypes.data_as(C.POINTER(C.c_double)), t.half_width,
                       int(t.subelements), t.pitch, t.center_frequency, t.fractional_bandwidth,
                       t.elevation_height, t.elevation_focus, t.elevation_core_weight,
                       t.elevation_tail_weight, t.elevation_aperture_factor), el


def plan_rf_chunks(t: Transducer, n_scatterers: int, medium: MediumParams, sampling_rate: float,
                   duration: float, budget: int) -> RfChunkPlan:
    """simulate.cpp:580-586 / plan_layout:389-416."""
    tc, keep = _td(t)
    out = RfChunkPlanC()
    check(load().fqfg_plan_rf_chunks(C.byref(tc), int(n_scatterers), C.byref(medium._c()),
                                     float(sampling_rate), float(duration), int(budget),
                                     C.byref(out)))
    return RfChunkPlan(out.blocks, out.block_scatterers, out.per_scatterer_bytes, out.fixed_bytes)


def _simulate(cloud, t, tx, medium, fs, duration, chunked, budget, stats):
    validate_transducer(t)
    pos = np.ascontiguousarray(np.asarray(cloud.positions, np.float64).reshape(-1, 3))
    refl = np.ascontiguousarray(np.asarray(cloud.reflectivity, np.float64).ravel())
    E = t.n_elements()
    if pos.shape[0] == 0:
        raise Error("scatterer cloud is empty")
    if refl.size != pos.shape[0]:
        raise Error("cloud reflectivity count does not match positions")
    delays = np.ascontiguousarray(
        np.asarray(tx.delays if tx.delays is not None else [], np.float64))
    apod = np.ascontiguousarray(
        np.asarray(tx.apodization if tx.apodization is not None else [], np.float64))
    if delays.size != E:
        raise Error("transmit delays do not match element count")
    if apod.size != E:
        raise Error("transmit apodization does not match element count")
    T = int(round(fs * duration)) if fs > 0 and duration > 0 else 16
    out = np.zeros((max(T, 16), E))
    tc, keep = _td(t)
    ns = C.c_int()
    st = RfSimStatsC()
    check(load().fqfg_simulate_rf(pos.ctypes.data, refl.ctypes.data, pos.shape[0], C.byref(tc),
                                  delays.ctypes.data, apod.ctypes.data, C.byref(medium._c()),
                                  float(fs), float(duration), int(chunked), int(budget),
                                  out.ctypes.data, C.byref(ns), C.byref(st)))
    if stats is not None:
        stats.blocks, stats.frequencies = st.blocks, st.frequencies
        stats.peak_tracked_bytes = st.peak_tracked_bytes
        stats.pair_bin_products = st.pair_bin_products
    return RfFrame(out[: ns.value].copy(), float(fs), 0.0, tx)


def simulate_rf(cloud: ScattererCloud, t: Transducer, tx: TxEvent, medium: MediumParams,
                sampling_rate: float, duration: float,
                stats: Optional[RfSimStats] = None) -> RfFrame:
    """simulate.cpp:588-597: errors if the pair geometry exceeds the medium's
    budget (use simulate_rf_chunked)."""
    return _simulate(cloud, t, tx, medium, sampling_rate, duration, 0, 0, stats)


def simulate_rf_chunked(cloud: ScattererCloud, t: Transducer, tx: TxEvent, medium: MediumParams,
                        sampling_rate: float, duration: float, budget: int,
                        stats: Optional[RfSimStats] = None) -> RfFrame:
    """simulate.cpp:599-606 (the budget sets the reported block plan)."""
    return _simulate(cloud, t, tx, medium, sampling_rate, duration, 1, budget, stats)


def compose_frames(tissue_frames: Sequence[ScattererCloud], flow_frames: Sequence[ScattererCloud],
                   static_tissue: bool, t: Transducer, tx: TxEvent, medium: MediumParams,
                   sampling_rate: float, duration: float,
                   stats: Optional[ComposeStats] = None) -> List[RfFrame]:
    """simulate.cpp:608-644: per-frame tissue echoes plus flow echoes; a
    static tissue cloud is simulated once and reused."""
    if len(flow_frames) == 0:
        raise Error("no flow frames to compose")
    if static_tissue:
        if len(tissue_frames) == 0:
            raise Error("static tissue requires one tissue cloud")
    elif len(tissue_frames) != len(flow_frames):
        raise Error("tissue and flow frame counts do not match")
    local = ComposeStats()
    T = int(round(sampling_rate * duration))

    def sim(cloud, kind):
        if cloud.size() == 0:
            validate_transducer(t)
            return RfFrame(np.zeros((T, t.n_elements())), float(sampling_rate), 0.0, tx)
        setattr(local, kind, getattr(local, kind) + 1)
        return simulate_rf_chunked(cloud, t, tx, medium, sampling_rate, duration,
                                   medium.scatterer_memory_budget)

    out = []
    tissue_rf = sim(tissue_frames[0], "tissue_simulations") if static_tissue else None
    for i, fl in enumerate(flow_frames):
        if not static_tissue:
            tissue_rf = sim(tissue_frames[i], "tissue_simulations")
        flow_rf = sim(fl, "flow_simulations")
        out.append(RfFrame(tissue_rf.samples + flow_rf.samples, float(sampling_rate), 0.0, tx))
    if stats is not None:
        stats.tissue_simulations = local.tissue_simulations
        stats.flow_simulations = local.flow_simulations
    return out
