"""Print PD rel-L2 and SSIM/PSNR (reference metrics) of the GPU chains vs the
reference chain on the phantom cases of tests/phantom_cases.py (GPU box)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_05464_b200 as P  # noqa: E402
from paper_2509_05464_b200 import pipeline as PL  # noqa: E402
from tests import phantom_cases as PC  # noqa: E402
from tests.golden_io import rel_l2  # noqa: E402

rows = []
for name in PC.CASES:
    c, ph = PC.case(name), PC.phantom(name)
    bf = P.BeamformParams(c=1540.0, center_frequency=c.fc, f_number=1.5)
    rec = PL.Reconstructor(c.fs, 0.0, c.angles, c.F, c.T, c.grid, c.elements, bf, keep_lo=c.lo,
                           keep_hi=c.F)
    pd = rec.step(torch.from_numpy(ph.rf).cuda()).pd.cpu().numpy()
    pd_ref, m_ref, gimg = PC.reference(name)
    m = PC.score(name, pd, gimg)
    rows.append({"case": name, "grid": list(c.grid.dims), "elements": len(c.elements),
                 "angles": len(c.angles), "frames": c.F, "band": [c.lo, c.F],
                 "pd_rel_l2": rel_l2(pd, pd_ref),
                 "gpu": {k: float(v) for k, v in m.items()},
                 "reference": {k: float(v) for k, v in m_ref.items()}})
    print(json.dumps(rows[-1]))
