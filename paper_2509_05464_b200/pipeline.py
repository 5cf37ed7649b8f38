"""Kernel-by-kernel RF -> power Doppler reconstruction over the device entry
points of the C ABI (run_beamform + run_post, proj/src/pipeline/run.cpp:397-487),
optionally depth-slab sharded over a torch.distributed process group.

The production host is the C++ reconstruction engine (fqfg_recon_*,
engine.Engine: ring-buffered RF streaming, cross-ensemble overlap, NCCL);
this module composes the same kernels one call at a time and is what the
engine's tests compare against bit for bit.  PyTorch supplies device memory,
the stream and the process group; every kernel is in libfqfgpu.so:

  demod + DAS   fqfg_das_dev      (rank's z-slab of voxels)
  Gram          fqfg_gram_dev     (rank's voxels)   -> all_reduce(sum)  [only collective]
  eigensolve    fqfg_eig_band_dev (replicated, deterministic; vectors the band needs)
  projection+PD fqfg_project_pd_dev (rank's voxels) -> gather PD slabs to rank 0

The slab split balances the DAS work (active aperture pairs per z-plane).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from ._native import Error, PlanInfo, check, load
from .beamform import BeamformParams, GridSpec, _desc, _probe


def active_pairs_per_plane(grid: GridSpec, elements: np.ndarray, f_number: float) -> np.ndarray:
    """Count of (voxel, element) pairs inside the receive aperture for each
    z-plane (das.cpp:165-168), used to balance depth slabs."""
    nx, ny, nz = grid.dims
    x = grid.origin[0] + np.arange(nx) * grid.spacing[0]
    y = grid.origin[1] + np.arange(ny) * grid.spacing[1]
    el = np.asarray(elements)
    out = np.zeros(nz)
    dx2 = (x[None, :] - el[:, 0:1]) ** 2  # [E][nx]
    for k in range(nz):
        z = grid.origin[2] + k * grid.spacing[2]
        if f_number <= 0:
            out[k] = nx * ny * len(el)
            continue
        lim = (z - el[:, 2]) / (2.0 * f_number)  # [E]
        rem = np.where(lim[:, None] >= 0, lim[:, None] ** 2 - dx2, -1.0)
        half = np.sqrt(np.maximum(rem, 0.0))
        lo = np.searchsorted(y, (el[:, 1:2] - half).ravel(), side="left").reshape(half.shape)
        hi = np.searchsorted(y, (el[:, 1:2] + half).ravel(), side="right").reshape(half.shape)
        out[k] = np.sum(np.where(rem >= 0, hi - lo, 0))
    return out


def slab_bounds(weights: np.ndarray, parts: int, align: int = 1) -> List[Tuple[int, int]]:
    """Split planes [0, nz) into `parts` contiguous slabs of near-equal weight,
    boundaries on multiples of `align`."""
    nz = len(weights)
    cum = np.concatenate([[0.0], np.cumsum(weights)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, parts):
        target = total * r / parts
        k = int(np.searchsorted(cum, target))
        k = int(round(k / align)) * align
        k = min(max(k, cuts[-1]), nz)
        cuts.append(k)
    cuts.append(nz)
    return [(cuts[i], cuts[i + 1]) for i in range(parts)]


class DasPlan:
    """fqfg_das_plan for one ensemble geometry on the current device."""

    def __init__(self, fs, t0, angles, n_frames, n_samples, grid: GridSpec, elements,
                 bp: BeamformParams):
        A = len(angles)
        E = np.asarray(elements).reshape(-1, 3).shape[0]
        self.desc, self._keep = _desc(n_frames, A, n_samples, E, fs, t0, angles)
        self.probe, self._el = _probe(elements)
        self._grid, self._bf = grid._c(), bp._c()
        self.grid, self.bp = grid, bp
        self.F, self.A, self.T, self.E = n_frames, A, n_samples, E
        self.handle = C.c_void_p()
        L = load()
        check(L.fqfg_das_plan_create(C.byref(self.desc), C.byref(self._grid),
                                     C.byref(self.probe), C.byref(self._bf),
                                     C.byref(self.handle)))
        info = PlanInfo()
        check(L.fqfg_das_plan_info_get(self.handle, C.byref(info)))
        self.n_points = int(info.n_points)
        self.frames_per_pass = int(info.frames_per_pass)
        self.n_passes = int(info.n_passes)
        self.work_bytes = int(info.work_bytes)
        self.active_pairs = int(info.active_pairs)
        self.tile = tuple(info.tile)
        self.tensor_cores = info.mode == 2  # das_tc (else das2)

    def close(self):
        if self.handle:
            load().fqfg_das_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, d_rf, k_begin, k_end, d_x, d_work, d_counters=None, stream=0):
        check(load().fqfg_das_dev(self.handle, d_rf, int(k_begin), int(k_end), d_x, d_work,
                                  d_counters, stream))


@dataclass
class StepResult:
    pd: object          # torch.float64 [N] on rank 0 (None elsewhere when sharded)
    sigma: object       # torch.float64 [F]


class Reconstructor:
    """RF [F][A][T][E] (device, f32) -> PD [N] (device, f64) for one geometry.

    ``group``: a torch.distributed process group for depth-slab sharding
    (None = single GPU).  ``shard=(rank, world)`` without a group builds one
    rank's slab on this device for tests that replay a sharded run on one GPU
    (the caller then does the Gram reduction; see das_gram / finish).
    Buffers are allocated once and reused per step."""

    def __init__(self, fs, t0, angles, n_frames, n_samples, grid: GridSpec, elements,
                 bp: BeamformParams, keep_lo=2, keep_hi=None, group=None, device=None,
                 shard=None):
        import torch
        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.plan = DasPlan(fs, t0, angles, n_frames, n_samples, grid, elements, bp)
        self.F, self.N = n_frames, grid.num_points()
        self.lo, self.hi = keep_lo, keep_hi if keep_hi is not None else n_frames
        if not (1 <= self.lo <= self.hi <= self.F):
            raise Error(f"retained band must satisfy 1 <= lo <= hi <= frames, got [{self.lo}, "
                        f"{self.hi}] with {self.F} frames")
        self.group = group
        self.rank, self.world = 0, 1
        if group is not None:
            import torch.distributed as dist
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        elif shard is not None:
            self.rank, self.world = int(shard[0]), int(shard[1])
        nx, ny, nz = grid.dims
        w = active_pairs_per_plane(grid, elements, bp.f_number)
        self._wplanes = w
        self.slabs = slab_bounds(w, self.world, align=self.plan.tile[2])
        self.k0, self.k1 = self.slabs[self.rank]
        self.v0, self.v1 = self.k0 * nx * ny, self.k1 * nx * ny
        self.active_pairs = self.plan.active_pairs
        F, N = self.F, self.N
        dev = self.device
        # X is [F][N]; a rank only writes/reads its slab's voxel range.
        self.x = torch.empty((F, N, 2), dtype=torch.float32, device=dev)
        self.work = torch.empty(max(self.plan.work_bytes, load().fqfg_gram_work_bytes(F)),
                                dtype=torch.uint8, device=dev)
        self.gram = torch.empty((F, F, 2), dtype=torch.float64, device=dev)
        self.w = torch.empty(F, dtype=torch.float64, device=dev)
        self.v = torch.empty((F, F, 2), dtype=torch.float64, device=dev)
        self.pd = torch.zeros(N, dtype=torch.float64, device=dev)
        # RF samples this rank's slab (the whole grid on one GPU) can read
        # (fqfg_das_slab_samples): the echoes before the earliest arrival any
        # voxel receives, and after the latest, never reach the output, so the
        # streamed paths upload [t_begin, t_end) only.
        tb, te = C.c_int(0), C.c_int(n_samples)
        if self.k1 > self.k0:
            check(load().fqfg_das_slab_samples(self.plan.handle, self.k0, self.k1, C.byref(tb),
                                               C.byref(te)))
        self.t_begin, self.t_end = tb.value, te.value

    def _stream(self, stream):
        if stream is not None:
            return stream
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def upload_rf(self, h_rf, d_rf, stream=None) -> int:
        """Pinned host RF [F][A][T][E] f32 -> device buffer of the same shape,
        copying only samples [t_begin, t_end) (what this rank's slab reads).
        Returns the bytes copied."""
        F, A, T, E = h_rf.shape
        row = E * 4
        nbytes = (self.t_end - self.t_begin) * row
        check(load().fqfg_copy_slices_h2d(d_rf.data_ptr(), h_rf.data_ptr(), F * A, T * row,
                                          self.t_begin * row, nbytes, self._stream(stream)))
        return F * A * nbytes

    def das_gram(self, d_rf, stream=None):
        """Demod + DAS of this rank's slab, then its partial Gram (self.gram)."""
        s = self._stream(stream)
        self.plan.run(d_rf.data_ptr(), self.k0, self.k1, self.x.data_ptr(), self.work.data_ptr(),
                      None, s)
        self._gram(s)

    def _gram(self, s):
        check(load().fqfg_gram_dev(self.x.data_ptr(), self.F, self.N, self.v0, self.v1,
                                   self.gram.data_ptr(), self.work.data_ptr(), s))

    def finish(self, stream=None):
        """Eigensolve of self.gram (already reduced) + projection + PD of this
        rank's voxels."""
        s = self._stream(stream)
        L = load()
        check(L.fqfg_eig_band_dev(self.gram.data_ptr(), self.F, self.lo, self.hi,
                                  self.w.data_ptr(), self.v.data_ptr(), s))
        check(L.fqfg_project_pd_dev(self.x.data_ptr(), self.F, self.N, self.v0, self.v1,
                                    self.v.data_ptr(), self.lo, self.hi, None,
                                    self.pd.data_ptr(), s))

    def step(self, d_rf, stream=None, das=None) -> StepResult:
        """One RF -> PD reconstruction; das (optional) enqueues this rank's
        demod + DAS into self.x in place of the one-call form."""
        torch = self.torch
        if das is None:
            self.das_gram(d_rf, stream)
        else:
            das()
            self._gram(self._stream(stream))
        if self.group is not None and self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.gram, group=self.group)
        self.finish(stream)
        pd = self.pd
        if self.group is not None and self.world > 1:
            pd = self.gather_pd()
        sigma = torch.sqrt(torch.clamp(self.w, min=0.0))
        return StepResult(pd, sigma)

    def gather_pd(self):
        nx, ny, _ = self.plan.grid.dims
        return gather_slabs(self.pd, self.slabs, nx * ny, self.group)


def gather_slabs(vec, slabs, plane, group):
    """Reassemble a voxel vector whose rank r holds only planes slabs[r] (a
    contiguous voxel range) on rank 0; other ranks get None."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sizes = [(k1 - k0) * plane for k0, k1 in slabs]
    v0 = slabs[rank][0] * plane
    buf = torch.zeros(max(sizes), dtype=vec.dtype, device=vec.device)
    buf[: sizes[rank]] = vec[v0:v0 + sizes[rank]]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return None
    return torch.cat([p[:n] for p, n in zip(parts, sizes)])
