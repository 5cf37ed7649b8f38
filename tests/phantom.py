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


def make_phantom(elements, fc, fs, angles, n_samples, n_frames, grid, seed=20260816,
                 n_tissue=1500, n_blood=500, blood_db=-20.0, radius=None, flow=0.02,
                 frame_rate=500.0, motion_peak=4e-3, c=1540.0, t0=0.0) -> Phantom:
    from paper_2509_05464_b200.phantom import FlowPhantom
    ph = FlowPhantom(grid, seed, n_tissue, n_blood, blood_db, radius, flow, frame_rate,
                     motion_peak)
    el = np.asarray(elements, np.float64).reshape(-1, 3)
    E = el.shape[0]
    sigma = 0.7 / (2 * np.pi * 0.7 * fc) * 2.0  # pulse envelope s.d. (s)
    K = int(np.ceil(4 * sigma * fs))
    T = n_samples
    rf = np.zeros((n_frames, len(angles), T, E), np.float64)
    blood_pos = []
    for f in range(n_frames):
        fr = ph.frame(f)
        tissue_f, blood_f = fr.tissue, fr.blood
        amp_t, amp_b = fr.tissue_refl, fr.blood_refl
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
