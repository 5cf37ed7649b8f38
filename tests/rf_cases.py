"""RF-synthesis fixtures shared by tests/golden/make_golden_rf.py (which
records the reference simulator's output for them) and the tests (which
rebuild the same inputs from the stored parameters)."""
import math

import numpy as np

import paper_2509_05464_b200 as P

RF_CASES = ["rfsim_small", "rfsim_lens", "rfsim_matrix", "rfsim_chunked", "rfsim_compose"]


def _small_probe(lens):
    # test_rf.cpp:31-43
    el = np.array([[(i - 1.0) * 0.4e-3, 0.0, 0.0] for i in range(3)])
    kw = dict(elevation_height=4e-3, elevation_focus=12e-3) if lens else {}
    return P.Transducer(el, "test", 0.4e-3, 5e6, half_width=0.15e-3, subelements=2,
                        fractional_bandwidth=0.5, **kw)


def _matrix8():
    el = np.array([[(i - 3.5) * 0.3e-3, (j - 3.5) * 0.3e-3, 0.0] for j in range(8)
                   for i in range(8)])
    return P.Transducer(el, "m8", 0.3e-3, 3e6, half_width=0.135e-3, subelements=2,
                        fractional_bandwidth=0.6)


def case_inputs(name):
    """(meta, transducer, tx event, inputs) of fixture `name`."""
    small_pos = [[1.0e-3, 0.3e-3, 8.0e-3], [-0.7e-3, 0.0, 11.0e-3], [0.2e-3, -0.2e-3, 9.5e-3]]
    small_refl = [1.0, -0.7, 0.35]
    if name in ("rfsim_small", "rfsim_lens"):
        td = _small_probe(name == "rfsim_lens")
        tx = P.plane_wave_delays(td, 3.0 * math.pi / 180.0, 1540.0)
        tx.apodization = np.array([1.0, 0.8, 1.2])
        meta = dict(fs=20e6, duration=20e-6, medium=dict(c=1540.0, att=0.7))
        return meta, td, tx, dict(positions=np.array(small_pos), reflectivity=np.array(small_refl))
    td = _matrix8()
    tx = P.plane_wave_delays(td, -4.0 * math.pi / 180.0, 1540.0)
    meta = dict(fs=12e6, duration=30e-6, medium=dict(c=1540.0, att=0.5))
    rng = np.random.default_rng(2509)
    if name in ("rfsim_matrix", "rfsim_chunked"):
        pos = np.stack([rng.uniform(-3e-3, 3e-3, 300), rng.uniform(-3e-3, 3e-3, 300),
                        rng.uniform(6e-3, 20e-3, 300)], 1)
        refl = rng.standard_normal(300)
        if name == "rfsim_chunked":
            meta.update(chunked=True, chunk_budget=1_357_440)
        return meta, td, tx, dict(positions=pos, reflectivity=refl)
    # rfsim_compose
    tpos = np.stack([rng.uniform(-3e-3, 3e-3, 40), rng.uniform(-3e-3, 3e-3, 40),
                     rng.uniform(6e-3, 20e-3, 40)], 1)
    trefl = rng.standard_normal(40)
    fpos0 = np.stack([rng.uniform(-1e-3, 1e-3, 6), np.zeros(6), rng.uniform(9e-3, 14e-3, 6)], 1)
    frefl = 0.1 * rng.standard_normal(6)
    flow = [(fpos0 + np.array([0.0, 0.0, 0.05e-3 * f]), frefl) for f in range(4)]
    meta["frames"] = 4
    return meta, td, tx, dict(tissue=[(tpos, trefl)], flow=flow)
