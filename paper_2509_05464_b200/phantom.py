"""A deterministic flow phantom as scatterer clouds (input generator for
parity tests and dataset generation; not part of the reference path).

Tissue speckle fills the grid's box (reflectivity N(0, 1)) outside a curved
vessel; blood scatterers (reflectivity 10^(blood_db / 20) N(0, 1), -20 dB by
default, config.hpp:73) fill the tube and are advected along its centreline
at `flow` m/s.  Optional rigid periodic tissue motion along z ("cardiac",
1.2 Hz, SURVEY 8(d) RF content modes).  frame(f) returns the clouds of frame
f; the blood positions also feed ground_truth_pd.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _centreline(u, lo, hi, two_d):
    """Curved vessel centreline through the box, u in [0, 1)."""
    mid, ext = (lo + hi) / 2, (hi - lo)
    x = lo[0] + 0.1 * ext[0] + 0.8 * ext[0] * u
    z = mid[2] + 0.22 * ext[2] * np.sin(2 * np.pi * 0.8 * u + 0.3)
    y = np.full_like(u, mid[1]) if two_d else mid[1] + 0.2 * ext[1] * np.cos(2 * np.pi * 0.6 * u)
    return np.stack([x, y, z], axis=-1)


@dataclass
class FlowFrame:
    tissue: np.ndarray        # [n_t][3]
    tissue_refl: np.ndarray   # [n_t]
    blood: np.ndarray         # [n_b][3]
    blood_refl: np.ndarray    # [n_b]


class FlowPhantom:
    def __init__(self, grid, seed=20260816, n_tissue=1500, n_blood=500, blood_db=-20.0,
                 radius=None, flow=0.02, frame_rate=500.0, motion_peak=4e-3):
        rng = np.random.default_rng(seed)
        dims, sp, org = np.asarray(grid.dims), np.asarray(grid.spacing), np.asarray(grid.origin)
        self.two_d = bool(dims[1] == 1)
        lo = org - 2 * sp
        hi = org + (dims - 1) * sp + 2 * sp
        if self.two_d:
            lo[1] = hi[1] = org[1]
        self.lo, self.hi = lo, hi
        ext = hi - lo
        self.radius = radius if radius is not None else 2.5 * sp[0]
        tis = lo + rng.random((n_tissue * 2, 3)) * ext
        cl = _centreline(np.linspace(0, 1, 400), lo, hi, self.two_d)
        d = np.min(np.linalg.norm(tis[:, None, :] - cl[None, :, :], axis=-1), axis=1)
        self.tissue = tis[d > self.radius][:n_tissue]
        self.tissue_refl = rng.standard_normal(len(self.tissue))
        self.length = np.sum(np.linalg.norm(np.diff(cl, axis=0), axis=1))
        self.u0 = rng.random(n_blood)
        self.r = self.radius * np.sqrt(rng.random(n_blood))
        self.th = 2 * np.pi * rng.random(n_blood)
        self.blood_refl = rng.standard_normal(n_blood) * 10 ** (blood_db / 20)
        self.flow, self.frame_rate, self.motion_peak = flow, frame_rate, motion_peak

    def frame(self, f: int) -> FlowFrame:
        t_f = f / self.frame_rate
        dz = self.motion_peak / (2 * np.pi * 1.2) * np.sin(2 * np.pi * 1.2 * t_f)
        shift = np.array([0.0, 0.0, dz])
        u = (self.u0 + self.flow * t_f / self.length) % 1.0
        lo, hi, two_d = self.lo, self.hi, self.two_d
        cpos = _centreline(u, lo, hi, two_d)
        du = 1e-4
        tang = _centreline(np.minimum(u + du, 1.0), lo, hi, two_d) - _centreline(
            np.maximum(u - du, 0.0), lo, hi, two_d)
        tang /= np.linalg.norm(tang, axis=1, keepdims=True)
        n = len(u)
        a1 = (np.cross(tang, [0.0, 1.0, 0.0]) if not two_d else np.tile([0.0, 0.0, 1.0], (n, 1)))
        a1 /= np.linalg.norm(a1, axis=1, keepdims=True) + 1e-30
        a2 = np.cross(tang, a1)
        off = (self.r * np.cos(self.th))[:, None] * a1
        if not two_d:
            off = off + (self.r * np.sin(self.th))[:, None] * a2
        return FlowFrame(self.tissue + shift, self.tissue_refl, cpos + off + shift,
                         self.blood_refl)
