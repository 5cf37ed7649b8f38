"""Tensor-core DAS time and K blocks per launch for voxel tiles of 64
(FQFG_DAS_SHAPE=13,2,16,8,TX,TY,TZ), e.g. python scripts/debug/tc_tiles.py C 4,8,2 8,8,1"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2509_05464_b200 import _native as N  # noqa: E402
from paper_2509_05464_b200.engine import Engine  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1]
w = W.config(cfg)
L = N.load()
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 7, 0))
for t in sys.argv[2:]:
    os.environ["FQFG_DAS_SHAPE"] = "13,2,16,8," + t
    eng = Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf())
    os.environ.pop("FQFG_DAS_SHAPE")
    eng.run_dev([d_rf])
    eng.set_timing(True)
    eng.run_dev([d_rf] * 2)
    dm, da, fl, tot = eng.last_timing()
    kb = eng.mma_blocks() / 2
    print(f"{cfg} tile {t}: DAS {da / 2:.1f} ms, step {tot / 2:.1f} ms, K blocks {kb:.3e}, "
          f"tile {tuple(eng.info.tile)}", flush=True)
    eng.close()
