"""Regenerate tests/golden/rfsim_*.npz from the REFERENCE's own RF simulator
(run in the build container, where /root/reference exists).

proj/src/rf/simulate.cpp includes <fftw3.h>; FFTW is absent from this image,
so oracle/Makefile compiles the file unmodified against oracle/fftw_stub (the
c2r transform by its published definition).  Fixtures:

  rfsim_small     test_rf.cpp:229-261's case: 3-element probe (v = 2, 5 MHz,
                  50 % bandwidth), 3 deg transmit with apodization (1, 0.8,
                  1.2), attenuation 0.7 dB/cm/MHz, three scatterers, 20 MHz, 20 us
  rfsim_lens      the same probe with a fixed elevation lens (the knot-
                  interpolated elevation factor)
  rfsim_matrix    an 8 x 8 matrix array at 3 MHz / 12 MHz, -4 deg, 300 seeded
                  scatterers, 30 us
  rfsim_chunked   rfsim_matrix through simulate_rf_chunked with a budget that
                  forces several scatterer blocks (RfSimStats.blocks > 1)
  rfsim_compose   compose_frames over 4 frames: static tissue (40 scatterers
                  simulated once) + moving flow (6 scatterers per frame)

Usage:  make -C oracle && python tests/golden/make_golden_rf.py
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402
from tests.rf_cases import RF_CASES, case_inputs  # noqa: E402


def main():
    # simulate_rf_chunked's block plan counts FQF_THREADS scratch buffers
    # (simulate.cpp:402-405): pinned to 8 so the fixture's RfSimStats do not
    # depend on the machine (the tests set the same value).
    os.environ["FQF_THREADS"] = "8"
    for name in RF_CASES:
        meta, td, tx, inp = case_inputs(name)
        med = meta["medium"]
        if name == "rfsim_compose":
            out, st = O.ref_compose_frames(inp["tissue"], inp["flow"], True, td, tx.delays,
                                           tx.apodization, angle=tx.angle, c=med["c"],
                                           att=med["att"], fs=meta["fs"],
                                           duration=meta["duration"])
        else:
            out, st = O.ref_simulate_rf(inp["positions"], inp["reflectivity"], td, tx.delays,
                                        tx.apodization, angle=tx.angle, c=med["c"],
                                        att=med["att"], fs=meta["fs"], duration=meta["duration"],
                                        chunked=meta.get("chunked", False),
                                        chunk_budget=meta.get("chunk_budget", 0))
        meta = dict(meta, stats=st)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), meta=json.dumps(meta), rf=out)
        print("wrote", name, out.shape, st)


if __name__ == "__main__":
    main()
