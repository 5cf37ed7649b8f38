"""One warm-up + one demod + DAS launch at a config's full size for ncu
(FQFG_DAS_SHAPE selects the kernel shape), e.g.

    ncu --set full -k regex:das2_kernel -s 1 -c 1 python scripts/profile_das.py C
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05464_b200 import _native as N  # noqa: E402
from paper_2509_05464_b200 import pipeline as PL  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402

w = W.config(sys.argv[1] if len(sys.argv) > 1 else "C")
L = N.load()
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 7, 0))
p = PL.DasPlan(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf())
work = torch.empty(p.work_bytes, dtype=torch.uint8, device="cuda")
x = torch.empty((w.n_frames, w.grid.num_points(), 2), dtype=torch.float32, device="cuda")
for _ in range(2):
    p.run(d_rf.data_ptr(), 0, w.grid.dims[2], x.data_ptr(), work.data_ptr())
torch.cuda.synchronize()
print("done", p.tile, p.frames_per_pass)
