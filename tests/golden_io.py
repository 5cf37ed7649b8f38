"""Load the golden fixtures in tests/golden (see tests/golden/make_golden.py)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def numpy_rf(seed, shape):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, size=shape).astype(np.float32).astype(np.float64)


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    if "rf" not in arrays and "rf_seed" in meta:
        arrays["rf"] = numpy_rf(meta["rf_seed"], tuple(meta["rf_shape"]))
    return meta, arrays


DAS_CASES = ["das_kat", "das_kat_nearest", "das_kat_fnum0", "das_partition", "das_identical",
             "das_linearity", "das_cached", "das_cached_off", "das_oow", "das_matrix32", "das_l11"]


def das_kwargs(meta):
    return dict(c=meta.get("c", 1540.0), fc=meta["fc"], f_number=meta.get("f_number", 1.5),
                interp_order=meta.get("interp_order", 1),
                lowpass_taps=meta.get("lowpass_taps", 33))


def rel_max(a, b):
    scale = max(np.abs(a).max(), np.abs(b).max())
    return 0.0 if scale == 0 else float(np.abs(a - b).max() / scale)


def rel_l2(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))
