"""Tensor-core DAS (FQFG_DAS_KERNEL=3) vs the default kernel on the small
workload: relative L2 / max deviation and DasStats.  Not a test (see
tests/test_gpu_parity.py::test_das_kernel_variants_agree)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_05464_b200 as P  # noqa: E402
from paper_2509_05464_b200 import workloads as W  # noqa: E402

w = W.small()
rf = np.random.default_rng(12).uniform(-1, 1, w.rf_shape()).astype(np.float32)
os.environ.pop("FQFG_DAS_KERNEL", None)
base, st0 = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf(),
                                    want_stats=True)
os.environ["FQFG_DAS_KERNEL"] = "3"
got, st1 = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf(),
                                   want_stats=True)
print(f"rel_l2 {np.linalg.norm(got - base) / np.linalg.norm(base):.3e} "
      f"rel_max {np.abs(got - base).max() / np.abs(base).max():.3e} stats_equal {st0 == st1}",
      flush=True)
