"""RF synthesis throughput (pair-bin products / s) for one plane-wave
transmit of the matrix32x32 probe at config-C timing (fs 12 MHz, 64 us),
GPU (fqfg_simulate_rf_dev, device-resident, CUDA events) vs the C engine
restatement (single thread) on a scatterer sample.  Never a bench.py number."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_05464_b200 as P  # noqa: E402
from paper_2509_05464_b200 import _native as N, rf  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
td = P.matrix32x32()
tx = P.plane_wave_delays(td, 4.0 * np.pi / 180.0, 1540.0)
med = rf.MediumParams()
fs, dur = 12e6, 64e-6
rng = np.random.default_rng(1)
pos = np.stack([rng.uniform(-16e-3, 16e-3, n), rng.uniform(-16e-3, 16e-3, n),
                rng.uniform(10e-3, 42e-3, n)], 1)
refl = rng.standard_normal(n)
tc, keep = rf._td(td)
L = N.load()
d_pos = torch.from_numpy(pos).cuda()
d_refl = torch.from_numpy(refl).cuda()
d_el = torch.from_numpy(np.ascontiguousarray(td.elements)).cuda()
d_del = torch.from_numpy(tx.delays).cuda()
d_apod = torch.from_numpy(tx.apodization).cuda()
T = int(round(fs * dur))
out = torch.empty((T, td.n_elements()), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def run():
    N.check(L.fqfg_simulate_rf_dev(d_pos.data_ptr(), d_refl.data_ptr(), n, C.byref(tc),
                                   d_el.data_ptr(), d_del.data_ptr(), d_apod.data_ptr(),
                                   C.byref(med._c()), fs, dur, out.data_ptr(), None, s))


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
_, lo, hi, _ = O.rf_passband(td, fs, dur)
bins = hi - lo + 1
pb = n * td.n_elements() * td.subelements * bins
# CPU: the engine restatement, single thread, on a 64-scatterer sample
ns = 64
t = time.perf_counter()
O.simulate_rf(pos[:ns], refl[:ns], td, tx.delays, tx.apodization, fs=fs, duration=dur)
cpu_s = time.perf_counter() - t
cpu_pb = ns * td.n_elements() * td.subelements * bins / cpu_s
print(json.dumps({"scatterers": n, "elements": td.n_elements(), "subelements": td.subelements,
                  "bins": bins, "T": T, "gpu_ms_per_transmit": ms,
                  "gpu_pair_bin_per_s": pb / (ms / 1e3),
                  "cpu_engine_1thread_pair_bin_per_s": cpu_pb, "cpu_sample_scatterers": ns}))
