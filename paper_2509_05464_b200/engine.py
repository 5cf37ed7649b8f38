"""Python face of the C++ reconstruction engine (fqfg_recon_*, csrc/recon.cu):
RF channel data -> power Doppler for a sequence of ensembles, one engine per
device / depth slab (run_beamform + run_post, proj/src/pipeline/run.cpp:397-487).

The engine owns its plan, buffers and streams; this wrapper only marshals
pointers (numpy / torch host buffers in, PD and singular values out).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import numpy as np

from ._native import ALLREDUCE_FN, Error, ReconInfo, ReconOpts, check, load
from .beamform import BeamformParams, GridSpec, _desc, _probe


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 makes it, every rank passes it)."""
    buf = C.create_string_buffer(128)
    check(load().fqfg_nccl_unique_id(buf))
    return buf.raw


def _ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    raise TypeError(f"expected a numpy array or torch tensor, got {type(a)}")


class Engine:
    """fqfg_recon for one ensemble geometry on the current CUDA device.

    rank / world: this process's depth slab; world > 1 needs ``nccl_id`` (the
    same bytes on every rank) or ``allreduce(dev_ptr, count, stream) -> int``
    (a stream-ordered sum of ``count`` doubles over the ranks)."""

    def __init__(self, fs, t0, angles, n_frames, n_samples, grid: GridSpec, elements,
                 bp: BeamformParams, keep_lo: int = 2, keep_hi: Optional[int] = None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 allreduce: Optional[Callable[[int, int, int], int]] = None,
                 device_budget: int = 0, ring_frames: int = 0, x_buffers: int = 0,
                 gram_fp64: bool = False, rf_broadcast: bool = False):
        A = len(angles)
        E = np.asarray(elements).reshape(-1, 3).shape[0]
        self.F, self.A, self.T, self.E = n_frames, A, n_samples, E
        self.grid = grid
        self.N = grid.num_points()
        self._desc, self._keep = _desc(n_frames, A, n_samples, E, fs, t0, angles)
        self._probe, self._el = _probe(elements)
        self._grid, self._bf = grid._c(), bp._c()
        o = ReconOpts()
        o.keep_lo, o.keep_hi = keep_lo, keep_hi or 0
        o.rank, o.world = rank, world
        self._id = None
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = C.cast(self._id, C.c_void_p)
        self._cb = None
        if allreduce is not None:
            self._cb = ALLREDUCE_FN(lambda user, ptr, n, stream: int(allreduce(ptr, n, stream)))
            o.allreduce = self._cb
        o.device_budget, o.ring_frames, o.x_buffers = device_budget, ring_frames, x_buffers
        o.gram_fp64 = int(bool(gram_fp64))
        o.rf_broadcast = int(bool(rf_broadcast))
        self._opts = o
        self.handle = C.c_void_p()
        check(load().fqfg_recon_create(C.byref(self._desc), C.byref(self._grid),
                                       C.byref(self._probe), C.byref(self._bf), C.byref(o),
                                       C.byref(self.handle)))

    @property
    def info(self) -> ReconInfo:
        info = ReconInfo()
        check(load().fqfg_recon_info_get(self.handle, C.byref(info)))
        return info

    def run(self, rf: Sequence, pd: Optional[Sequence] = None,
            sigma: Optional[Sequence] = None) -> None:
        """rf[k]: host [F][A][T][E] f32 (numpy or pinned torch); pd[k]: host
        [N] f64 (written: every voxel on rank 0 of an NCCL run, this rank's
        voxels otherwise); sigma[k]: host [F] f64."""
        n = len(rf)
        for a in rf:
            if a is None:  # a broadcast receiver (rf_broadcast, rank > 0)
                continue
            if tuple(a.shape) != (self.F, self.A, self.T, self.E):
                raise Error(f"RF shape {tuple(a.shape)} != {(self.F, self.A, self.T, self.E)}")
        rfp = (C.c_void_p * max(n, 1))(*[None if a is None else _ptr(a) for a in rf])
        pdp = (C.c_void_p * max(n, 1))(*[_ptr(a) for a in pd]) if pd is not None else None
        sgp = (C.c_void_p * max(n, 1))(*[_ptr(a) for a in sigma]) if sigma is not None else None
        check(load().fqfg_recon_run(self.handle, n, rfp, pdp, sgp))

    def run_dev(self, d_rf: Sequence, d_pd=None) -> None:
        """Device-resident RF d_rf[k] (torch CUDA [F][A][T][E] f32), read in
        place; the last ensemble's PD -> d_pd (torch CUDA [N] f64)."""
        n = len(d_rf)
        rfp = (C.c_void_p * max(n, 1))(*[_ptr(a) for a in d_rf])
        check(load().fqfg_recon_run_dev(self.handle, n, rfp,
                                        _ptr(d_pd) if d_pd is not None else None))

    def copy_iq(self, v_begin: Optional[int] = None, v_end: Optional[int] = None) -> np.ndarray:
        """IQ (the DAS output) of the last ensemble reconstructed, voxels
        [v_begin, v_end) of this engine's slab: complex64 [F][v_end - v_begin]."""
        info = self.info
        v_begin = info.v_begin if v_begin is None else v_begin
        v_end = info.v_end if v_end is None else v_end
        out = np.empty((self.F, v_end - v_begin), dtype=np.complex64)
        check(load().fqfg_recon_copy_iq(self.handle, v_begin, v_end, out.ctypes.data))
        return out

    def report(self):
        """(singular values [F], mode correlation [F][F]) of the last
        ensemble: SvdReport (svd.cpp:49-76) from the resident IQ."""
        s = np.zeros(self.F)
        c = np.zeros((self.F, self.F))
        check(load().fqfg_recon_report(self.handle, s.ctypes.data, c.ctypes.data))
        return s, c

    def set_timing(self, on: bool) -> None:
        check(load().fqfg_recon_set_timing(self.handle, int(bool(on))))

    def last_timing(self):
        """(demod_ms, das_ms, filter_ms, total_ms) of the last timed run: the
        spans summed over its ensembles, and the whole run."""
        a, b, c, t = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        check(load().fqfg_recon_last_timing(self.handle, C.byref(a), C.byref(b), C.byref(c),
                                            C.byref(t)))
        return a.value, b.value, c.value, t.value

    def mma_blocks(self) -> int:
        """Tensor-core DAS K blocks issued by the last run (0 with das2)."""
        n = C.c_ulonglong()
        check(load().fqfg_recon_mma_blocks(self.handle, C.byref(n)))
        return int(n.value)

    def close(self) -> None:
        if self.handle:
            load().fqfg_recon_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
