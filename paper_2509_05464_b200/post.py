"""fqf::post on the B200: svd_filter (post/svd.hpp:23-25, svd.cpp:29-93) and
power_doppler (post/render.hpp:13, render.cpp:23-42) over the C ABI.

svd_filter: Casorati matrix X (voxels x frames), X = U S V^H, output
U_b S_b V_b^H = X V_b V_b^H for the 1-based band keep_lo..keep_hi.  On the GPU:
FP64 Gram X^H X, on-device FP64 Jacobi eigensolve (V, S^2), then the band
projection with power Doppler fused into its epilogue.  SvdReport carries the
singular spectrum and mode_correlation, the Pearson correlation of the |U|
columns (svd.cpp:55-75), computed on the GPU from |X V| / sigma.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

import ctypes as C

from ._native import Error, check, load
from .beamform import GridSpec, IqVolume

__all__ = ["SvdReport", "VoxelGrid", "svd_filter", "svd_filter_array", "power_doppler",
           "power_doppler_array", "DbScale", "render_db", "bmode", "mip", "ground_truth_pd",
           "MetricsReport", "metrics", "metrics_csv", "metrics_json"]


@dataclass
class SvdReport:
    """svd.hpp:10-16."""
    singular_values: List[float] = field(default_factory=list)
    mode_correlation: List[float] = field(default_factory=list)
    n_modes: int = 0
    keep_lo: int = 0
    keep_hi: int = 0


@dataclass
class VoxelGrid:
    """The scalar VoxelGrid power_doppler returns (core/grid.hpp:16-84)."""
    dims: tuple
    spacing: tuple
    origin: tuple
    data: np.ndarray


def _check_ensemble(ensemble: Sequence[IqVolume]):
    if len(ensemble) == 0:
        raise Error("svd_filter needs a nonempty ensemble")
    first = ensemble[0]
    n = first.grid.num_points()
    if n <= 0:
        raise Error("svd_filter needs a nonempty grid")
    for fr in ensemble:
        if tuple(fr.grid.dims) != tuple(first.grid.dims):
            raise Error("ensemble frames must share one grid")
        if fr.values.size != n:
            raise Error("frame value count must match the grid")
    if len(ensemble) < 2:
        raise Error("svd_filter needs at least two frames")
    if len(ensemble) > n:
        raise Error("svd_filter needs at least as many voxels as frames")
    return n


def svd_filter_array(x: np.ndarray, keep_lo: int, keep_hi: int, want_filtered=True,
                     want_pd=False, want_corr=False):
    """x [F][N] complex -> (filtered [F][N] complex64 | None, sigma [F], pd [N] | None)
    or, with want_corr, a 4-tuple ending in the [F][F] mode correlation."""
    x = np.ascontiguousarray(x, dtype=np.complex64)
    F, N = x.shape
    out = np.empty((F, N), np.complex64) if want_filtered else None
    sigma = np.zeros(F)
    pd = np.zeros(N) if want_pd else None
    corr = np.zeros((F, F)) if want_corr else None
    check(load().fqfg_svd_filter(x.ctypes.data, F, N, keep_lo, keep_hi,
                                 out.ctypes.data if out is not None else None, sigma.ctypes.data,
                                 pd.ctypes.data if pd is not None else None,
                                 corr.ctypes.data if corr is not None else None))
    if want_corr:
        return out, sigma, pd, corr
    return out, sigma, pd


def svd_filter(ensemble: Sequence[IqVolume], keep_lo: int, keep_hi: int,
               report: Optional[SvdReport] = None) -> List[IqVolume]:
    n = _check_ensemble(ensemble)
    F = len(ensemble)
    if not (1 <= keep_lo <= keep_hi <= F):
        raise Error(f"retained band must satisfy 1 <= lo <= hi <= frames, got [{keep_lo}, "
                    f"{keep_hi}] with {F} frames")
    x = np.stack([np.asarray(fr.values) for fr in ensemble])
    y, sigma, _, corr = svd_filter_array(x, keep_lo, keep_hi, want_corr=True) if report \
        is not None else svd_filter_array(x, keep_lo, keep_hi) + (None,)
    if report is not None:
        report.n_modes = F
        report.keep_lo = keep_lo
        report.keep_hi = keep_hi
        report.singular_values = [float(s) for s in sigma]
        report.mode_correlation = [float(c) for c in corr.ravel()]
    return [IqVolume(fr.grid, fr.frame_index, fr.n_angles, y[f].astype(np.complex128))
            for f, fr in enumerate(ensemble)]


def power_doppler_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex64)
    F, N = x.shape
    pd = np.zeros(N)
    check(load().fqfg_power_doppler(x.ctypes.data, F, N, pd.ctypes.data))
    return pd


def power_doppler(ensemble: Sequence[IqVolume]) -> VoxelGrid:
    if len(ensemble) == 0:
        raise Error("power_doppler needs at least one frame")
    first = ensemble[0]
    n = first.grid.num_points()
    if n <= 0:
        raise Error("power_doppler needs a nonempty grid")
    for fr in ensemble:
        if tuple(fr.grid.dims) != tuple(first.grid.dims):
            raise Error("ensemble frames must share one grid")
        if fr.values.size != n:
            raise Error("frame value count must match the grid")
    pd = power_doppler_array(np.stack([np.asarray(fr.values) for fr in ensemble]))
    g: GridSpec = first.grid
    return VoxelGrid(tuple(g.dims), tuple(g.spacing), tuple(g.origin), pd)


# ------------------------------------------------ display and scoring --
# post/render.hpp:15-40 and post/metrics.hpp:9-29, computed on the GPU
# (csrc/display.cu).

class DbScale:
    """render.hpp:15."""
    amplitude = 0  # 20 log10
    power = 1      # 10 log10


def _dims(v: VoxelGrid):
    return (C.c_int * 3)(*[int(d) for d in v.dims])


def _like(v: VoxelGrid, data, dims=None):
    return VoxelGrid(tuple(dims or v.dims), tuple(v.spacing), tuple(v.origin), data)


def render_db(volume: VoxelGrid, dynamic_range_db: float, scale: int) -> VoxelGrid:
    """render.cpp:44-68: dB re the peak, clipped to [-dr, 0], mapped to [0, 1]."""
    x = np.ascontiguousarray(volume.data, dtype=np.float64).ravel()
    if x.size == 0:
        raise Error("render_db needs a nonempty volume")
    out = np.empty_like(x)
    check(load().fqfg_render_db(x.ctypes.data, _dims(volume), float(dynamic_range_db),
                                1 if scale == DbScale.power else 0, out.ctypes.data))
    return _like(volume, out)


def bmode(iq: IqVolume, dynamic_range_db: float = 75.0) -> VoxelGrid:
    """render.cpp:70-78: |IQ| log-compressed (amplitude)."""
    g = iq.grid
    v = np.ascontiguousarray(np.asarray(iq.values, dtype=np.complex128).ravel())
    if v.size != g.num_points() or v.size == 0:
        raise Error("bmode needs an IQ volume matching its grid")
    out = np.empty(v.size)
    check(load().fqfg_bmode(v.ctypes.data, (C.c_int * 3)(*g.dims), float(dynamic_range_db),
                            out.ctypes.data))
    return VoxelGrid(tuple(g.dims), tuple(g.spacing), tuple(g.origin), out)


def mip(volume: VoxelGrid, axis: int) -> VoxelGrid:
    """render.cpp:80-104: maximum intensity projection along axis."""
    x = np.ascontiguousarray(volume.data, dtype=np.float64).ravel()
    dims = list(volume.dims)
    if not (0 <= axis < 3):
        raise Error(f"mip axis must be 0, 1, or 2, got {axis}")
    if x.size == 0:
        raise Error("mip needs a nonempty volume")
    out_dims = list(dims)
    out_dims[axis] = 1
    out = np.empty(int(np.prod(out_dims)))
    check(load().fqfg_mip(x.ctypes.data, _dims(volume), int(axis), out.ctypes.data))
    return _like(volume, out, out_dims)


def ground_truth_pd(positions_per_frame, grid: GridSpec, sigma_voxels: float) -> VoxelGrid:
    """render.cpp:106-145: Gaussian-splatted blood occupancy, peak-normalised."""
    frames = [np.asarray(p, dtype=np.float64).reshape(-1, 3) for p in positions_per_frame]
    if not frames:
        raise Error("ground_truth_pd needs at least one frame")
    counts = (C.c_int * len(frames))(*[len(f) for f in frames])
    xyz = np.ascontiguousarray(np.concatenate(frames)) if frames else np.zeros((0, 3))
    out = np.empty(max(grid.num_points(), 0))
    gc = grid._c()
    check(load().fqfg_ground_truth_pd(xyz.ctypes.data, counts, len(frames), C.byref(gc),
                                      float(sigma_voxels), out.ctypes.data))
    return VoxelGrid(tuple(grid.dims), tuple(grid.spacing), tuple(grid.origin), out)


@dataclass
class MetricsReport:
    """metrics.hpp:9-13."""
    mse: float = 0.0
    psnr: float = 0.0
    ssim: float = 0.0


def metrics(test: VoxelGrid, reference: VoxelGrid) -> MetricsReport:
    """metrics.cpp:84-101: MSE, PSNR (unit peak), mean local SSIM."""
    if tuple(test.dims) != tuple(reference.dims):
        raise Error("metrics needs images of identical shape")
    a = np.ascontiguousarray(test.data, dtype=np.float64).ravel()
    b = np.ascontiguousarray(reference.data, dtype=np.float64).ravel()
    if a.size == 0:
        raise Error("metrics needs nonempty images")
    out = np.zeros(3)
    check(load().fqfg_metrics(a.ctypes.data, b.ctypes.data, _dims(test), out.ctypes.data))
    return MetricsReport(float(out[0]), float(out[1]), float(out[2]))


def metrics_csv(r: MetricsReport) -> str:
    """metrics.cpp:114-119 (17 significant digits)."""
    return f"{r.mse:.17g},{'inf' if np.isinf(r.psnr) else format(r.psnr, '.17g')},{r.ssim:.17g}\n"


def metrics_json(r: MetricsReport) -> str:
    """metrics.cpp:121-126."""
    psnr = '"inf"' if np.isinf(r.psnr) else format(r.psnr, ".17g")
    return f'{{"mse": {r.mse:.17g}, "psnr": {psnr}, "ssim": {r.ssim:.17g}}}\n'
