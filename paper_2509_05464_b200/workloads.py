"""The benchmark configurations of BASELINE.json as concrete synthetic inputs
(probe, f_c/fs, angles, grid, T, F).

Common parameters: c = 1540 m/s, F# = 1.5, 33 low-pass taps, linear
interpolation, t0 = 0 (das.hpp:76-82 defaults); fs = 4 f_c (config.cpp:471-474).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .beamform import BeamformParams, GridSpec

DEG = math.pi / 180.0


@dataclass
class Workload:
    name: str
    elements: np.ndarray  # [E][3]
    fc: float
    fs: float
    angles: np.ndarray    # radians
    grid: GridSpec
    n_samples: int
    n_frames: int
    ensembles: int = 1

    @property
    def n_elements(self):
        return self.elements.shape[0]

    @property
    def n_angles(self):
        return len(self.angles)

    def bf(self) -> BeamformParams:
        return BeamformParams(c=1540.0, center_frequency=self.fc, f_number=1.5, interp_order=1,
                              lowpass_taps=33)

    def nominal_samples(self) -> int:
        """voxel x element x angle x frame (the BASELINE metric's unit)."""
        return self.grid.num_points() * self.n_elements * self.n_angles * self.n_frames

    def rf_shape(self):
        return (self.n_frames, self.n_angles, self.n_samples, self.n_elements)

    def describe(self):
        g = self.grid
        return {"workload": self.name, "probe_elements": self.n_elements,
                "angles": self.n_angles, "voxels": list(g.dims), "samples_T": self.n_samples,
                "frames": self.n_frames, "f_c_hz": self.fc, "fs_hz": self.fs}


def matrix_probe(n: int, pitch: float = 0.3e-3) -> np.ndarray:
    """n x n matrix, j outer / i inner (transducer.cpp:54-58)."""
    h = (n - 1) / 2.0
    return np.array([[(i - h) * pitch, (j - h) * pitch, 0.0] for j in range(n) for i in range(n)])


def linear_probe(n: int = 128, pitch: float = 0.3e-3) -> np.ndarray:
    h = (n - 1) / 2.0
    return np.array([[(i - h) * pitch, 0.0, 0.0] for i in range(n)])


def _centered(n, s):
    return -(n - 1) * s / 2.0


def config(name: str) -> Workload:
    name = name.upper()
    if name == "A":
        return Workload("A: l11-4v 128 el, 3 angles, 256x1x256 px, 50 frames", linear_probe(128),
                        7.7e6, 30.8e6, np.array([-5, 0, 5]) * DEG,
                        GridSpec((256, 1, 256), (0.1e-3, 0.1e-3, 0.1e-3), (-12.75e-3, 0.0, 5e-3)),
                        1602, 50)
    sp = 0.2567e-3
    if name == "B":
        return Workload("B: matrix 32x32, 9 angles, 64^3 voxels, 100 frames", matrix_probe(32),
                        3e6, 12e6, np.arange(-8, 9, 2) * DEG,
                        GridSpec((64, 64, 64), (sp, sp, sp),
                                 (_centered(64, sp), _centered(64, sp), 10e-3)), 504, 100)
    if name in ("C", "E"):
        w = Workload("C: matrix 32x32, 9 angles, 128^3 voxels, 200 frames", matrix_probe(32),
                     3e6, 12e6, np.arange(-8, 9, 2) * DEG,
                     GridSpec((128, 128, 128), (sp, sp, sp),
                              (_centered(128, sp), _centered(128, sp), 10e-3)), 768, 200)
        if name == "E":
            w.name = "E: 100 ensembles of C"
            w.ensembles = 100
        return w
    if name == "D":
        return Workload("D: matrix 64x64, 15 angles, 256x256x192 voxels, 400 frames",
                        matrix_probe(64), 3e6, 12e6, np.arange(-14, 15, 2) * DEG,
                        GridSpec((256, 256, 192), (sp, sp, sp),
                                 (_centered(256, sp), _centered(256, sp), 10e-3)), 1176, 400)
    raise ValueError(f"unknown workload {name!r} (A-E)")


def small(name: str = "S") -> Workload:
    """A seconds-sized matrix-array case for smoke tests and the CPU oracle."""
    sp = 0.2567e-3
    return Workload("S: matrix 32x32, 3 angles, 8x6x4 voxels, 20 frames", matrix_probe(32), 3e6,
                    12e6, np.array([-4, 0, 4]) * DEG,
                    GridSpec((8, 6, 4), (sp, sp, sp), (-1.0e-3, -0.7e-3, 10e-3)), 224, 20)
