"""Deterministic flow phantom -> plane-wave RF, for image-quality parity tests.

Test infrastructure (input generator only): the GPU path and the reference
chain consume the SAME RF, so this is not a restatement of the reference's
frequency-domain simulator (proj/src/rf/simulate.cpp, needs FFTW); it is a
time-domain point-scatterer echo model with the reference's geometry
conventions:

* transmit delay of plane wave a: (x sin a + z cos a - min_e x_e sin a) / c
  (das.cpp:143-145, 162), receive |p - e| / c, echo at t = t_tx + t_rx;
* pulse: Gaussian-modulated cosine at f_c (fractional bandwidth ~70 %);
* tissue: uniform speckle, reflectivity N(0, 1), rigid periodic motion along
  z ("cardiac", 1.2 Hz, SURVEY 8(d) RF content modes);
* blood: scatterers in a curved tube, reflectivity 10^(-20/20) relative to
  tissue (config.hpp:73), flowing along the centreline; their positions per
  frame feed the reference's ground_truth_pd (render.cpp:106-145).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np


@dataclass
class Phantom:
    rf: np.ndarray                 # [F][A][T][E] float32
    blood: List[np.ndarray] = field(default_factory=list)  # per frame [n][3] positions (m)


def _centreline(u, box_lo, box_hi, two_d):
    """Curved vessel centreline through the box, u in [0, 1)."""
    lo, hi = np.asarray(box_lo), np.asarray(box_hi)
    mid, ext = (lo + hi) / 2, (hi - lo)
    x = lo[0] + 0.1 * ext[0] + 0.8 * ext[0] * u
    z = mid[2] + 0.22 * ext[2] * np.sin(2 * np.pi * 0.8 * u + 0.3)
    y = np.full_like(u, mid[1]) if two_d else mid[1] + 0.2 * ext[1] * np.cos(2 * np.pi * 0.6 * u)
    return np.stack([x, y, z], axis=-1)


def make_phantom(elements, fc, fs, angles, n_samples, n_frames, grid, seed=20260816,
                 n_tissue=1500, n_blood=500, blood_db=-20.0, radius=None, flow=0.02,
                 frame_rate=500.0, motion_peak=4e-3, c=1540.0, t0=0.0) -> Phantom:
    rng = np.random.default_rng(seed)
    el = np.asarray(elements, np.float64).reshape(-1, 3)
    E = el.shape[0]
    dims, sp, org = np.asarray(grid.dims), np.asarray(grid.spacing), np.asarray(grid.origin)
    two_d = dims[1] == 1
    lo = org - 2 * sp
    hi = org + (dims - 1) * sp + 2 * sp
    if two_d:
        lo[1] = hi[1] = org[1]
    ext = hi - lo
    radius = radius if radius is not None else 2.5 * sp[0]

    # Tissue speckle outside the vessel.
    tis = lo + rng.random((n_tissue * 2, 3)) * ext
    cl = _centreline(np.linspace(0, 1, 400), lo, hi, two_d)
    d = np.min(np.linalg.norm(tis[:, None, :] - cl[None, :, :], axis=-1), axis=1)
    tis = tis[d > radius][:n_tissue]
    amp_t = rng.standard_normal(len(tis))

    # Blood: tube coordinates (u along, radial offset), advected by `flow` m/s.
    length = np.sum(np.linalg.norm(np.diff(cl, axis=0), axis=1))
    u0 = rng.random(n_blood)
    r = radius * np.sqrt(rng.random(n_blood))
    th = 2 * np.pi * rng.random(n_blood)
    amp_b = rng.standard_normal(n_blood) * 10 ** (blood_db / 20)

    sigma = 0.7 / (2 * np.pi * 0.7 * fc) * 2.0  # pulse envelope s.d. (s)
    K = int(np.ceil(4 * sigma * fs))
    T = n_samples
    rf = np.zeros((n_frames, len(angles), T, E), np.float64)
    blood_pos = []
    for f in range(n_frames):
        t_f = f / frame_rate
        dz = motion_peak / (2 * np.pi * 1.2) * np.sin(2 * np.pi * 1.2 * t_f)
        tissue_f = tis + np.array([0.0, 0.0, dz])
        u = (u0 + flow * t_f / length) % 1.0
        cpos = _centreline(u, lo, hi, two_d)
        du = 1e-4
        tang = _centreline(np.minimum(u + du, 1.0), lo, hi, two_d) - _centreline(
            np.maximum(u - du, 0.0), lo, hi, two_d)
        tang /= np.linalg.norm(tang, axis=1, keepdims=True)
        a1 = np.cross(tang, [0.0, 1.0, 0.0]) if not two_d else np.tile([0.0, 0.0, 1.0], (n_blood, 1))
        a1 /= np.linalg.norm(a1, axis=1, keepdims=True) + 1e-30
        a2 = np.cross(tang, a1)
        off = (r * np.cos(th))[:, None] * a1 + (0 if two_d else (r * np.sin(th))[:, None] * a2)
        blood_f = cpos + off
        blood_f = blood_f + np.array([0.0, 0.0, dz])
        blood_pos.append(blood_f)
        pos = np.concatenate([tissue_f, blood_f])
        amp = np.concatenate([amp_t, amp_b])
        rx = np.linalg.norm(pos[:, None, :] - el[None, :, :], axis=-1) / c  # [S][E]
        for a, ang in enumerate(angles):
            sa, ca = np.sin(ang), np.cos(ang)
            ref = np.min(el[:, 0] * sa)
            tau = (pos[:, 0] * sa + pos[:, 2] * ca - ref) / c  # [S]
            s = (tau[:, None] + rx - t0) * fs                 # [S][E] sample position
            base = np.floor(s).astype(np.int64)
            acc = np.zeros(T * E)
            col = np.arange(E)[None, :]
            for k in range(-K, K + 1):
                idx = base + k
                dt = (idx - s) / fs
                val = amp[:, None] * np.exp(-0.5 * (dt / sigma) ** 2) * np.cos(2 * np.pi * fc * dt)
                ok = (idx >= 0) & (idx < T)
                acc += np.bincount((idx * E + col)[ok], weights=val[ok], minlength=T * E)
            rf[f, a] = acc.reshape(T, E)
    return Phantom(rf.astype(np.float32), blood_pos)
