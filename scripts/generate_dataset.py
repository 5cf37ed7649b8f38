"""End-to-end on one GPU: flow phantom -> RF ensemble (GPU simulator) ->
demod + DAS + SVD filter + PD (pipeline.Reconstructor) -> rendered PD scored
against the rendered ground truth (GPU render_db / ground_truth_pd / metrics),
the reference pipeline's run_beamform + run_post + run_metrics chain
(run.cpp:397-506) for one dataset item.  Prints one JSON line of timings and
scores.  Static tissue (simulated once per angle), blood flowing at 2 cm/s.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_05464_b200 as P  # noqa: E402
from paper_2509_05464_b200 import dataset, pipeline, post, rf  # noqa: E402
from paper_2509_05464_b200.phantom import FlowPhantom  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--voxels", type=int, default=48)
ap.add_argument("--frames", type=int, default=40)
ap.add_argument("--angles", type=int, default=5)
ap.add_argument("--tissue", type=int, default=20000)
ap.add_argument("--blood", type=int, default=2000)
ap.add_argument("--lo", type=int, default=3)
a = ap.parse_args()

td = P.matrix32x32()
sp = 0.2567e-3
n = a.voxels
grid = P.GridSpec((n, n, n), (sp, sp, sp), (-(n - 1) * sp / 2, -(n - 1) * sp / 2, 10e-3))
angles = np.linspace(-8, 8, a.angles) * np.pi / 180
fs, fc = 12e6, td.center_frequency
zmax = grid.origin[2] + (n - 1) * sp + 1e-3
duration = (2 * np.sqrt(zmax ** 2 + 2 * (6e-3) ** 2) / 1540.0) * 1.15
duration = np.ceil(duration * fs) / fs
ph = FlowPhantom(grid, seed=7, n_tissue=a.tissue, n_blood=a.blood, motion_peak=0.0)
med = rf.MediumParams()

torch.cuda.synchronize()
t0 = time.perf_counter()
d_rf = dataset.simulate_ensemble(ph, td, angles, med, fs, duration, a.frames)
torch.cuda.synchronize()
t_rf = time.perf_counter() - t0

T = d_rf.shape[2]
bf = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=1.5)
rec = pipeline.Reconstructor(fs, 0.0, angles, a.frames, T, grid, td.elements, bf, keep_lo=a.lo,
                             keep_hi=a.frames)
rec.step(d_rf)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = rec.step(d_rf)
torch.cuda.synchronize()
t_rec = time.perf_counter() - t0

pd = out.pd.cpu().numpy()
gt = post.ground_truth_pd([ph.frame(f).blood for f in range(a.frames)], grid, 1.0)
img = post.render_db(post.VoxelGrid(grid.dims, grid.spacing, grid.origin, pd), 60.0,
                     post.DbScale.power)
gimg = post.render_db(gt, 60.0, post.DbScale.power)
m = post.metrics(img, gimg)
inside = pd[gt.data > 0.3].mean() / pd[gt.data < 0.01].mean()
print(json.dumps({"voxels": [n, n, n], "frames": a.frames, "angles": a.angles,
                  "samples_T": int(T), "tissue_scatterers": a.tissue,
                  "blood_scatterers": a.blood, "band": [a.lo, a.frames],
                  "rf_synthesis_s": t_rf, "transmits": a.frames * a.angles,
                  "reconstruction_s": t_rec, "pd_in_vessel_over_outside": float(inside),
                  "ssim": m.ssim, "psnr": m.psnr}))
