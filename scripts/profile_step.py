"""Warm-up + one RF -> PD step through the C++ engine (fqfg_recon_run_dev) at
a config's full size, for ncu launch lists:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python scripts/profile_step.py C
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05464_b200 import _native as N  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402
from paper_2509_05464_b200.engine import Engine  # noqa: E402

w = W.config(sys.argv[1] if len(sys.argv) > 1 else "C")
L = N.load()
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 7, 0))
eng = Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf())
eng.run_dev([d_rf])  # warm-up
eng.run_dev([d_rf])  # the profiled step
torch.cuda.synchronize()
print("done", tuple(eng.info.shape), eng.info.mode)
