"""A seconds-sized reconstruction for compute-sanitizer (racecheck /
synccheck / memcheck) of the production kernels: fused demodulation,
das2_kernel (default shape and the config-C shape: mbarrier pipeline, TMA
bulk copies, named barriers, setmaxnreg), the tensor-core Gram (TMA tensor
maps, tcgen05.mma / commit / ld, TMEM alloc), eigensolve, projection + PD.

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_05464_b200 as P  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402
from paper_2509_05464_b200.engine import Engine  # noqa: E402


def main():
    import torch
    torch.cuda.set_device(0)
    sp = 0.2567e-3
    w = W.Workload("san", W.matrix_probe(8), 3e6, 12e6, np.array([-4, 0, 4]) * W.DEG,
                   P.GridSpec((8, 8, 4), (sp, sp, sp), (-1e-3, -1e-3, 6e-3)), 160, 24)
    rf = np.random.default_rng(1).uniform(-1, 1, w.rf_shape()).astype(np.float32)
    for shape in (None, "13,2,16,8,4,8,2"):
        if shape:
            os.environ["FQFG_DAS_SHAPE"] = shape
        for fp64 in (False, True):
            eng = Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf(),
                         gram_fp64=fp64, device_budget=2 << 30)
            pd = np.zeros(w.grid.num_points())
            eng.run([rf], [pd])
            assert np.all(np.isfinite(pd)) and pd.max() > 0
            eng.close()
    print("sanitize case done")


if __name__ == "__main__":
    main()
