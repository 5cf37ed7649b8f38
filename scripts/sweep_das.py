"""Time demod + DAS (fqfg_das_dev) for das2_kernel shapes / lane mappings at a
config's full size: FQFG_DAS_SHAPE=J,VPW,NW,PW[,TX,TY,TZ] per plan (das2:
FQFG_DAS_TC=0 for the whole run),
interleaved A/B repeats, CUDA events; prints DAS ms per launch and checks the
variants agree bitwise with the first.

    FQFG_DAS_TC=0 python scripts/sweep_das.py C "13,2,16,8,4,8,2" "13,2,16,8,8,4,2"
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05464_b200 import _native as N  # noqa: E402
from paper_2509_05464_b200 import pipeline as PL  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402


def main():
    cfg = sys.argv[1]
    shapes = sys.argv[2:]
    reps = int(os.environ.get("REPS", "2"))
    w = W.config(cfg)
    L = N.load()
    d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
    N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 7, 0))
    plans = []
    for shape in shapes:
        os.environ["FQFG_DAS_SHAPE"] = shape
        plans.append(PL.DasPlan(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements,
                                w.bf()))
        os.environ.pop("FQFG_DAS_SHAPE", None)
    work = torch.empty(max(p.work_bytes for p in plans), dtype=torch.uint8, device="cuda")
    N_ = w.grid.num_points()
    xs = [torch.empty((w.n_frames, N_, 2), dtype=torch.float32, device="cuda") for _ in plans]
    times = {sh: [] for sh in shapes}
    for r in range(reps + 1):
        for sh, p, x in zip(shapes, plans, xs):
            L.fqfg_das_plan_set_timing(p.handle, 1)
            p.run(d_rf.data_ptr(), 0, w.grid.dims[2], x.data_ptr(), work.data_ptr())
            dm, da = C.c_double(), C.c_double()
            N.check(L.fqfg_das_last_timing(p.handle, C.byref(dm), C.byref(da)))
            L.fqfg_das_plan_set_timing(p.handle, 0)
            if r > 0:
                times[sh].append(da.value)
    for sh, x in zip(shapes, xs):
        same = bool(torch.equal(x, xs[0]))
        print(f"{cfg} shape {sh}: DAS {min(times[sh]):.1f} ms (runs {['%.1f' % t for t in times[sh]]})"
              f", bitwise equal to first: {same}", flush=True)


if __name__ == "__main__":
    main()
