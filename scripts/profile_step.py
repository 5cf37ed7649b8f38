"""One warm-up + N RF -> PD steps of a workload (for ncu launch lists and
captures; never a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_05464_b200 import _native as N, pipeline as PL, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="B")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--frames", type=int, default=0)
a = ap.parse_args()
w = W.config(a.config)
if a.frames:
    w.n_frames = a.frames
F, A, T, E = w.rf_shape()
rec = PL.Reconstructor(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf())
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
N.check(N.load().fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 1, 0))
for _ in range(1 + a.steps):
    rec.step(d_rf)
torch.cuda.synchronize()
print("ok", w.name, "tile", rec.plan.tile, "fpass", rec.plan.frames_per_pass,
      "passes", rec.plan.n_passes)
