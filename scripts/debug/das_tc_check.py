"""Tensor-core DAS (default) vs das2 (FQFG_DAS_TC=0) on one config: relative error and
DAS time (CUDA events) of each, e.g.  python scripts/debug/das_tc_check.py S B C
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2509_05464_b200 import _native as N  # noqa: E402
from paper_2509_05464_b200 import pipeline as PL  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402


def plan(w, tc):
    os.environ["FQFG_DAS_TC"] = "1" if tc else "0"
    p = PL.DasPlan(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf())
    os.environ.pop("FQFG_DAS_TC", None)
    return p


def run(L, p, w, d_rf, reps):
    work = torch.zeros(p.work_bytes, dtype=torch.uint8, device="cuda")
    x = torch.zeros((w.n_frames, w.grid.num_points(), 2), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    ts = []
    for r in range(reps):
        L.fqfg_das_plan_set_timing(p.handle, 1)
        p.run(d_rf.data_ptr(), 0, w.grid.dims[2], x.data_ptr(), work.data_ptr(),
              cnt.data_ptr() if r == 0 else None)
        dm, da = C.c_double(), C.c_double()
        N.check(L.fqfg_das_last_timing(p.handle, C.byref(dm), C.byref(da)))
        L.fqfg_das_plan_set_timing(p.handle, 0)
        ts.append((dm.value, da.value))
    torch.cuda.synchronize()
    return x, cnt.cpu().tolist(), ts


def main():
    L = N.load()
    for cfg in sys.argv[1:]:
        w = W.small() if cfg == "S" else W.config(cfg)
        d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
        N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 7, 0))
        reps = 1 if cfg == "S" else 3
        x0, c0, t0 = run(L, plan(w, False), w, d_rf, reps)
        x1, c1, t1 = run(L, plan(w, True), w, d_rf, reps)
        d = (x1 - x0).double()
        rel = float(d.norm() / x0.double().norm())
        mx = float(d.abs().max() / x0.double().abs().max())
        print(f"{cfg}: rel_l2 {rel:.3e} rel_max {mx:.3e} nan {bool(torch.isnan(x1).any())} "
              f"counters das2 {c0} tc {c1} | das2 demod/das ms {t0[-1][0]:.2f}/{t0[-1][1]:.2f} "
              f"tc {t1[-1][0]:.2f}/{t1[-1][1]:.2f}", flush=True)


if __name__ == "__main__":
    main()
