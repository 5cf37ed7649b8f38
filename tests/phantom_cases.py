"""Phantom cases for the image-quality parity tests (PD rel-L2
plus SSIM/PSNR of the rendered PD identical to 3 decimals), and the
reference chain they are judged against:

  IQ  = the reference's own das_reconstruct (oracle/_ref, FP64)
  SVD = the FP64 restatement of svd_filter (Eigen is absent; oracle/)
  PD  = the reference's power_doppler; images = its render_db (60 dB, power)
  GT  = the reference's ground_truth_pd over the blood scatterer tracks,
        metrics = its metrics() (run.cpp:457-492 does exactly this).
"""
from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np

from oracle import oracle as O
from paper_2509_05464_b200 import GridSpec
from paper_2509_05464_b200 import workloads as W
from tests.phantom import make_phantom

DR_DB = 60.0
GT_SIGMA = 1.0


@dataclass
class Case:
    name: str
    elements: np.ndarray
    fc: float
    fs: float
    angles: np.ndarray
    grid: GridSpec
    T: int
    F: int
    lo: int          # retained band [lo, F]: tissue motion needs more than rank 1


def case(name):
    if name == "linear2d":
        sp = 0.3e-3
        return Case(name, W.linear_probe(64, 0.3e-3), 5e6, 20e6, np.array([-5, 0, 5]) * W.DEG,
                    GridSpec((64, 1, 64), (sp, sp, sp), (-9.45e-3, 0.0, 6e-3)), 1000, 24, 6)
    if name == "matrix3d":
        sp = 0.2567e-3
        return Case(name, W.matrix_probe(12), 3e6, 12e6, np.array([-4, 0, 4]) * W.DEG,
                    GridSpec((24, 24, 24), (sp, sp, sp), (-2.95e-3, -2.95e-3, 8e-3)), 280, 20, 5)
    raise KeyError(name)


CASES = ["linear2d", "matrix3d"]


@functools.lru_cache(maxsize=None)
def phantom(name):
    c = case(name)
    return make_phantom(c.elements, c.fc, c.fs, c.angles, c.T, c.F, c.grid)


@functools.lru_cache(maxsize=None)
def reference(name):
    """(pd, metrics, gt_image) of the reference chain."""
    c, ph = case(name), phantom(name)
    g = c.grid
    iq, _ = O.ref_das(ph.rf.astype(np.float64), c.fs, 0.0, c.angles, c.elements, g.dims,
                      g.spacing, g.origin, fc=c.fc)
    y, _, _ = O.svd_filter(iq, c.lo, c.F)
    pd = O.ref_power_doppler(y, g.dims)
    gt = O.ref_ground_truth_pd(ph.blood, g.dims, g.spacing, g.origin, GT_SIGMA)
    gimg = O.ref_render_db(gt, g.dims, DR_DB, True)
    return pd, score(name, pd, gimg), gimg


def score(name, pd, gimg):
    g = case(name).grid
    return O.ref_metrics(O.ref_render_db(pd, g.dims, DR_DB, True), gimg, g.dims)
