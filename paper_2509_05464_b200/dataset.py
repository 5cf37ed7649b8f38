"""Dataset generation on the GPU: flow phantom -> plane-wave RF ensemble
(the reference's frequency-domain simulator, csrc/rfsim.cu) resident in HBM
as the [F][A][T][E] f32 input of the reconstruction (pipeline.Reconstructor).

Composition follows compose_frames (simulate.cpp:608-644): per frame and
angle, tissue echoes plus blood echoes summed in FP64 and rounded to f32 (the
RF container precision, simulate.cpp:638); with static tissue the tissue
response of each angle is simulated once and reused.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import check, load
from .beamform import Transducer, plane_wave_delays
from .phantom import FlowPhantom
from .rf import MediumParams, _td


def simulate_ensemble(phantom: FlowPhantom, t: Transducer, angles, medium: MediumParams,
                      fs: float, duration: float, n_frames: int, static_tissue: bool = True,
                      device=None):
    """RF [n_frames][A][T][E] float32 on the device (a torch tensor)."""
    import torch
    dev = device or torch.device("cuda", torch.cuda.current_device())
    L = load()
    tc, keep = _td(t)
    med = medium._c()
    s = torch.cuda.current_stream(dev).cuda_stream
    A, E = len(angles), t.n_elements()
    T = int(round(fs * duration))
    d_el = torch.from_numpy(np.ascontiguousarray(np.asarray(t.elements, np.float64))).to(dev)
    txs = [plane_wave_delays(t, float(a), medium.c) for a in angles]
    d_del = [torch.from_numpy(np.ascontiguousarray(x.delays)).to(dev) for x in txs]
    d_apod = [torch.from_numpy(np.ascontiguousarray(x.apodization)).to(dev) for x in txs]
    out = torch.empty((n_frames, A, T, E), dtype=torch.float32, device=dev)
    acc = torch.empty((T, E), dtype=torch.float64, device=dev)
    tis = torch.empty((A, T, E), dtype=torch.float64, device=dev)

    def sim(pos, refl, a, dst64):
        if len(pos) == 0:
            dst64.zero_()
            return
        dp = torch.from_numpy(np.ascontiguousarray(pos, np.float64)).to(dev)
        dr = torch.from_numpy(np.ascontiguousarray(refl, np.float64)).to(dev)
        check(L.fqfg_simulate_rf_dev(dp.data_ptr(), dr.data_ptr(), len(pos), C.byref(tc),
                                     d_el.data_ptr(), d_del[a].data_ptr(), d_apod[a].data_ptr(),
                                     C.byref(med), float(fs), float(duration), None,
                                     dst64.data_ptr(), s))

    for f in range(n_frames):
        fr = phantom.frame(f)
        for a in range(A):
            if f == 0 or not static_tissue:
                sim(fr.tissue, fr.tissue_refl, a, tis[a])
            sim(fr.blood, fr.blood_refl, a, acc)
            out[f, a].copy_(tis[a] + acc)
    return out
