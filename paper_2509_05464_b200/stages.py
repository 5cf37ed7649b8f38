"""GPU bodies of the reference pipeline's beamform / post / metrics stages
(proj/src/pipeline/run.cpp:397-507) over the same stage-directory layout and
with byte-compatible outputs, so a run directory produced by `fqflow run`
can be continued here and vice versa:

  rf/frame_FFFF_tx_AA.fqf       RF frames (simulate.cpp:629-658)       -> run_beamform
  beamform/Frame_<f+1>.fqf      IQ volumes, c128 (das.cpp:395-407)     -> run_post
  particles/frame_FFFF.fqf      particle tracks (hemo/particles.cpp:64-95)
  post/{bmode,pd,gt}.{fqf,pgm}  f64 grids (grid.cpp:79-99) + P5 graymaps (render.cpp:147-175)
  post/svd_report.json          nlohmann dump(2) of the SvdReport (run.cpp:470-485)
  metrics/metrics.{csv,json}    (run.cpp:489-507)

The stage configuration is the subset of the reference's RunConfig these
stages read (StageConfig; config parsing, manifests, content-hash caching and
locking are the reference's control plane and out of scope).
`run_beamform_post` is the fused GPU path: RF frames -> PD without the
IQ-volume round trip through the file system (still writing the frames the
reference's post stage would read when `write_frames` is set).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import fqf1, post
from .beamform import (BeamformParams, DasOptions, GridSpec, IqVolume, RfFrame, Transducer,
                       TxEvent, das_reconstruct, read_iq_volume)
from ._native import Error

__all__ = ["StageConfig", "rf_frame_rel", "iq_frame_rel", "particle_frame_rel", "write_rf_frame",
           "read_rf_frame", "write_particle_frame", "read_particle_frame", "write_grid",
           "read_grid", "write_pgm", "svd_report_json", "run_beamform", "run_post",
           "run_metrics", "run_beamform_post"]


@dataclass
class StageConfig:
    """The RunConfig fields run_beamform / run_post read (run.cpp:397-487)."""
    transducer: Transducer
    grid: GridSpec
    n_frames: int
    angles_deg: Sequence[float]
    sound_speed: float = 1540.0
    f_number: float = 1.5
    lowpass_taps: int = 33
    memory_budget_bytes: int = 100_000_000
    matrix_budget_bytes: int = 512_000_000
    cache_matrices: bool = True
    bmode_dynamic_range_db: float = 60.0
    pd_dynamic_range_db: float = 60.0
    svd_lo: int = 2
    svd_hi: int = 0               # 0 = n_frames (run.cpp:457)
    ground_truth_sigma_voxels: float = 1.0


# ------------------------------------------------------------------ paths --

def rf_frame_rel(f: int, a: int) -> str:
    """run.cpp:86-88."""
    return f"rf/frame_{f:04d}_tx_{a:02d}.fqf"


def iq_frame_rel(f: int) -> str:
    """run.cpp:89."""
    return f"beamform/Frame_{f + 1}.fqf"


def particle_frame_rel(f: int) -> str:
    """run.cpp:84."""
    return f"particles/frame_{f:04d}.fqf"


# --------------------------------------------------------------- file I/O --

def write_rf_frame(path: str, frame: RfFrame, frame_index: int) -> None:
    """simulate.cpp:629-640 (payload narrowed to f32)."""
    T, E = frame.samples.shape
    fqf1.write_container(path, [
        ("kind", "rf"), ("samples", str(T)), ("elements", str(E)),
        ("sampling_rate", fqf1.fmt17(frame.sampling_rate)), ("t0", fqf1.fmt17(frame.t0)),
        ("angle", fqf1.fmt17(frame.tx.angle)), ("frame", str(frame_index))],
        np.asarray(frame.samples, dtype=np.float32))


def read_rf_frame(path: str):
    """simulate.cpp:642-658 -> (RfFrame, frame index)."""
    h, payload = fqf1.read_container(path)
    hv = lambda k: fqf1.header_value(h, k)  # noqa: E731
    if hv("kind") != "rf":
        raise Error(f"{path}: not an rf frame container")
    T, E = int(hv("samples")), int(hv("elements"))
    x = fqf1.as_float64(payload)
    if x.size != T * E:
        raise Error(f"{path}: sample count does not match header dimensions")
    fr = RfFrame(x.reshape(T, E), float(hv("sampling_rate")), float(hv("t0")),
                 TxEvent(angle=float(hv("angle"))))
    return fr, int(hv("frame"))


def _cpp_default(x: float) -> str:
    """ostream << double at the default precision 6 (%g)."""
    return format(float(x), "g")


def write_particle_frame(path: str, positions: np.ndarray, frame_index: int,
                         time_s: float) -> None:
    """hemo/particles.cpp:64-79."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    fqf1.write_container(path, [("kind", "particles"), ("frame", str(frame_index)),
                                ("time", _cpp_default(time_s)), ("particles", str(len(pos)))],
                         pos.reshape(-1))


def read_particle_frame(path: str):
    """hemo/particles.cpp:81-95 -> (positions [n][3], frame index, time)."""
    h, payload = fqf1.read_container(path)
    hv = lambda k: fqf1.header_value(h, k)  # noqa: E731
    if hv("kind") != "particles":
        raise Error(f"{path}: not a particle container")
    flat = fqf1.as_float64(payload)
    if flat.size % 3:
        raise Error(f"{path}: particle payload is not 3 doubles per point")
    return flat.reshape(-1, 3), int(hv("frame")), float(hv("time"))


def write_grid(path: str, g: post.VoxelGrid, dtype: str = "f64") -> None:
    """grid.cpp:79-99 (scalar grids, f64 payload unless stated)."""
    d = [int(v) for v in g.dims]
    data = np.asarray(g.data, dtype=np.float64).reshape(-1)
    fqf1.write_container(path, [
        ("kind", "grid"), ("dims", f"{d[0]} {d[1]} {d[2]}"),
        ("spacing", " ".join(fqf1.fmt17(v) for v in g.spacing)),
        ("origin", " ".join(fqf1.fmt17(v) for v in g.origin)), ("components", "1")],
        data if dtype == "f64" else data.astype(np.float32))


def read_grid(path: str) -> post.VoxelGrid:
    """grid.cpp:101-121."""
    h, payload = fqf1.read_container(path)
    hv = lambda k: fqf1.header_value(h, k)  # noqa: E731
    if hv("kind") != "grid":
        raise Error(f"{path}: not a grid container")
    dims = tuple(int(v) for v in hv("dims").split())
    if int(hv("components")) != 1:
        raise Error(f"{path}: only scalar grids are supported here")
    data = fqf1.as_float64(payload)
    if data.size != dims[0] * dims[1] * dims[2]:
        raise Error(f"{path}: payload count does not match dims")
    return post.VoxelGrid(dims, tuple(float(v) for v in hv("spacing").split()),
                          tuple(float(v) for v in hv("origin").split()), data)


def write_pgm(path: str, img: post.VoxelGrid) -> None:
    """render.cpp:147-175: the first two non-singleton axes (then singleton
    axes) as columns u / rows v, values clamped to [0, 1], x 255 rounded half
    away from zero (std::lround) to 8 bits."""
    dims = [int(v) for v in img.dims]
    data = np.asarray(img.data, dtype=np.float64).reshape(-1)
    if data.size == 0:
        raise Error("write_pgm needs a nonempty image")
    axes = [ax for ax in range(3) if dims[ax] > 1][:2]
    if len(axes) == 2 and dims[3 - axes[0] - axes[1]] != 1:
        raise Error(f"write_pgm needs an image with a singleton axis, got dims "
                    f"{dims[0]}x{dims[1]}x{dims[2]}")
    for ax in range(3):
        if len(axes) < 2 and dims[ax] == 1 and (not axes or axes[0] != ax):
            axes.append(ax)
    u, v = axes
    vol = data.reshape(dims[2], dims[1], dims[0]).transpose(2, 1, 0)  # [x][y][z]
    sl = [0, 0, 0]
    sl[u] = slice(None)
    sl[v] = slice(None)
    plane = vol[tuple(sl)]
    img2 = plane.T if u < v else plane  # [row v][col u]
    x = np.clip(img2, 0.0, 1.0) * 255.0
    r = np.floor(x)
    byte = (r + (x - r >= 0.5)).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{dims[u]} {dims[v]}\n255\n".encode())
        f.write(np.ascontiguousarray(byte).tobytes())


def _json_number(x: float) -> str:
    """nlohmann::json's double output (dtoa_impl::format_buffer with
    min_exp = -4, max_exp = 15 over the shortest round-trip digits: fixed
    notation, '.0' on integral values, else d.ddde+XX; non-finite -> null)."""
    x = float(x)
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    r = repr(abs(x))
    mant, _, ex = r.partition("e")
    ip, _, fp = mant.partition(".")
    allds = (ip + fp).lstrip("0")
    n = len(allds) + (int(ex) if ex else 0) - len(fp)  # value = 0.DIGITS x 10^n
    digits = allds.rstrip("0")
    k = len(digits)
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        s = digits[0] + ("." + digits[1:] if k > 1 else "") + ("e+" if e >= 0 else "e-") + \
            f"{abs(e):02d}"
    return ("-" if x < 0 else "") + s


def svd_report_json(rep: post.SvdReport) -> str:
    """run.cpp:470-482: keys sorted (nlohmann object), dump(2) + newline."""
    def arr(xs, ind, num):
        if len(xs) == 0:
            return "[]"
        pad = " " * (ind + 2)
        return "[\n" + ",\n".join(pad + num(v) for v in xs) + "\n" + " " * ind + "]"
    fields = [("keep", arr([rep.keep_lo, rep.keep_hi], 2, lambda v: str(int(v)))),
              ("mode_correlation", arr(list(rep.mode_correlation), 2, _json_number)),
              ("n_modes", str(int(rep.n_modes))),
              ("singular_values", arr(list(rep.singular_values), 2, _json_number))]
    return "{\n" + ",\n".join(f'  "{k}": {v}' for k, v in fields) + "\n}\n"


# ----------------------------------------------------------------- stages --

def _bf(cfg: StageConfig) -> BeamformParams:
    return BeamformParams(c=cfg.sound_speed, center_frequency=cfg.transducer.center_frequency,
                          f_number=cfg.f_number, lowpass_taps=cfg.lowpass_taps)


def _read_rf(out: str, cfg: StageConfig):
    frames = []
    for f in range(cfg.n_frames):
        row = []
        for a in range(len(cfg.angles_deg)):
            p = os.path.join(out, rf_frame_rel(f, a))
            fr, idx = read_rf_frame(p)
            if idx != f:
                raise Error(f"{p}: header frame index {idx} does not match {f}")
            row.append(fr)
        frames.append(row)
    return frames


def run_beamform(out: str, cfg: StageConfig) -> List[str]:
    """run.cpp:397-431: RF frames -> das_reconstruct on the GPU -> the
    beamform/Frame_i.fqf volumes (write_frames, chunk files removed)."""
    frames = _read_rf(out, cfg)
    os.makedirs(os.path.join(out, "beamform"), exist_ok=True)
    opts = DasOptions(memory_budget_bytes=cfg.memory_budget_bytes,
                      matrix_budget_bytes=cfg.matrix_budget_bytes,
                      cache_matrices=cfg.cache_matrices, work_dir=os.path.join(out, "beamform"),
                      write_frames=True, keep_chunk_files=False)
    das_reconstruct(frames, cfg.grid, cfg.transducer, _bf(cfg), opts)
    return [iq_frame_rel(f) for f in range(cfg.n_frames)]


def _save_image(out: str, img: post.VoxelGrid, stem: str, outputs: List[str]) -> None:
    write_grid(os.path.join(out, "post", stem + ".fqf"), img)
    outputs.append(f"post/{stem}.fqf")
    d = img.dims
    flat = img if (d[0] == 1 or d[1] == 1 or d[2] == 1) else post.mip(img, 1)
    write_pgm(os.path.join(out, "post", stem + ".pgm"), flat)
    outputs.append(f"post/{stem}.pgm")


def _post_from(out: str, cfg: StageConfig, ensemble: Sequence[IqVolume]) -> List[str]:
    os.makedirs(os.path.join(out, "post"), exist_ok=True)
    outputs: List[str] = []
    _save_image(out, post.bmode(ensemble[0], cfg.bmode_dynamic_range_db), "bmode", outputs)
    hi = cfg.n_frames if cfg.svd_hi == 0 else cfg.svd_hi
    rep = post.SvdReport()
    filtered = post.svd_filter(ensemble, cfg.svd_lo, hi, rep)
    pd = post.power_doppler(filtered)
    _save_image(out, post.render_db(pd, cfg.pd_dynamic_range_db, post.DbScale.power), "pd",
                outputs)
    tracks = [read_particle_frame(os.path.join(out, particle_frame_rel(f)))[0]
              for f in range(cfg.n_frames)]
    gt = post.ground_truth_pd(tracks, ensemble[0].grid, cfg.ground_truth_sigma_voxels)
    _save_image(out, post.render_db(gt, cfg.pd_dynamic_range_db, post.DbScale.power), "gt",
                outputs)
    with open(os.path.join(out, "post", "svd_report.json"), "w") as f:
        f.write(svd_report_json(rep))
    outputs.append("post/svd_report.json")
    return outputs


def run_post(out: str, cfg: StageConfig) -> List[str]:
    """run.cpp:433-487: IQ volumes -> B-mode, SVD filter + PD (GPU), ground
    truth, SVD report."""
    ensemble = [read_iq_volume(os.path.join(out, iq_frame_rel(f))) for f in range(cfg.n_frames)]
    return _post_from(out, cfg, ensemble)


def run_beamform_post(out: str, cfg: StageConfig, write_frames: bool = True) -> List[str]:
    """Both stages with the ensemble kept in memory between them (no re-read
    of the F IQ volumes, run.cpp:438-440); outputs identical to run_beamform
    followed by run_post."""
    frames = _read_rf(out, cfg)
    opts = DasOptions(memory_budget_bytes=cfg.memory_budget_bytes,
                      matrix_budget_bytes=cfg.matrix_budget_bytes,
                      cache_matrices=cfg.cache_matrices,
                      work_dir=os.path.join(out, "beamform") if write_frames else "",
                      write_frames=write_frames, keep_chunk_files=False)
    if write_frames:
        os.makedirs(os.path.join(out, "beamform"), exist_ok=True)
    ensemble = das_reconstruct(frames, cfg.grid, cfg.transducer, _bf(cfg), opts)
    outputs = [iq_frame_rel(f) for f in range(cfg.n_frames)] if write_frames else []
    return outputs + _post_from(out, cfg, ensemble)


def run_metrics(out: str) -> List[str]:
    """run.cpp:489-507: SSIM / PSNR of the displayed PD against the ground truth."""
    pd = read_grid(os.path.join(out, "post", "pd.fqf"))
    gt = read_grid(os.path.join(out, "post", "gt.fqf"))
    rep = post.metrics(pd, gt)
    os.makedirs(os.path.join(out, "metrics"), exist_ok=True)
    with open(os.path.join(out, "metrics", "metrics.csv"), "w") as f:
        f.write(post.metrics_csv(rep))
    with open(os.path.join(out, "metrics", "metrics.json"), "w") as f:
        f.write(post.metrics_json(rep))
    return ["metrics/metrics.csv", "metrics/metrics.json"]


def stage_paths(cfg: StageConfig) -> Optional[dict]:
    """The relative paths each stage reads and writes (for callers that
    cache by content, as run.cpp's manifests do)."""
    A = len(cfg.angles_deg)
    return {"beamform": {"in": [rf_frame_rel(f, a) for f in range(cfg.n_frames)
                                for a in range(A)],
                         "out": [iq_frame_rel(f) for f in range(cfg.n_frames)]},
            "post": {"in": [iq_frame_rel(f) for f in range(cfg.n_frames)] +
                     [particle_frame_rel(f) for f in range(cfg.n_frames)],
                     "out": ["post/bmode.fqf", "post/bmode.pgm", "post/pd.fqf", "post/pd.pgm",
                             "post/gt.fqf", "post/gt.pgm", "post/svd_report.json"]},
            "metrics": {"in": ["post/pd.fqf", "post/gt.fqf"],
                        "out": ["metrics/metrics.csv", "metrics/metrics.json"]}}
