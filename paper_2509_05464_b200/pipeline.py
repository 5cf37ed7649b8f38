"""Device-resident RF -> power Doppler reconstruction (run_beamform + run_post,
proj/src/pipeline/run.cpp:397-487, fused and kept in HBM), optionally
depth-slab sharded over the ranks of a torch.distributed process group.

One process per GPU.  PyTorch supplies device memory, the stream and the
process group; every kernel is in libfqfgpu.so:

  demod + DAS   fqfg_das_dev      (rank's z-slab of voxels)
  Gram          fqfg_gram_dev     (rank's voxels)   -> all_reduce(sum)  [only collective]
  eigensolve    fqfg_eig_band_dev (replicated, deterministic; vectors the band needs)
  projection+PD fqfg_project_pd_dev (rank's voxels) -> gather PD slabs to rank 0

The slab split balances the DAS work (active aperture pairs per z-plane).
"""
from __future__ import annotations

import ctypes as C
import os
import math
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

    def _overlap_state(self):
        """Second set of filter buffers and a post-processing stream (single
        GPU): ensemble k's Gram / eigensolve / projection run on stream B while
        ensemble k+1's demod + DAS run on the working stream (the eigensolve
        is one CTA for ~14 ms at F = 200, the rest of the GPU would idle)."""
        torch = self.torch
        if hasattr(self, "_post"):
            return
        F, N, dev = self.F, self.N, self.device
        self._post = torch.cuda.Stream(dev)
        self._xb = [self.x, torch.empty_like(self.x)]
        self._gb = [self.gram, torch.empty_like(self.gram)]
        self._wb = [self.w, torch.empty_like(self.w)]
        self._vb = [self.v, torch.empty_like(self.v)]
        self._pdb = [self.pd, torch.empty_like(self.pd)]
        self._gwork = torch.empty(load().fqfg_gram_work_bytes(F), dtype=torch.uint8, device=dev)
        self._das_done = [torch.cuda.Event() for _ in range(2)]
        self._post_done = [torch.cuda.Event() for _ in range(2)]
        cur = torch.cuda.current_stream(dev)
        for e in self._post_done:
            e.record(cur)

    def _lead_slabs(self, fracs=(1 / 64, 1 / 16, 3 / 16, 1 / 2)):
        """Depth sub-slabs of this rank's planes for the first streamed
        ensemble, shallow to deep, each with the RF rows it needs:
        [(kb, ke, t_lo, t_hi)] with t_lo / t_hi cumulative (each slab's rows
        are uploaded on top of the previous ones).  Cuts at the plane fractions
        `fracs`: the first slab is thin (even the top planes read ~1/4 of the
        record, so its wait is that upload), each later one several times the
        last, so its DAS outlasts the upload of the next slab's rows
        (profiles/r01_stream_lead.md: one streamed ensemble at C 704 ms with 8
        equal slabs each demodulating all its rows, 674 ms with these cuts,
        incremental demodulation and a stream per sub-slab DAS)."""
        if hasattr(self, "_lead"):
            return self._lead
        n, al = self.k1 - self.k0, self.plan.tile[2]
        cuts = [0]
        for f in fracs:
            c = int(round(n * f / al)) * al
            if cuts[-1] < c < n:
                cuts.append(c)
        cuts.append(n)
        lead, hi = [], self.t_begin
        for kb, ke in zip(cuts[:-1], cuts[1:]):
            kb, ke = kb + self.k0, ke + self.k0
            if ke <= kb:
                continue
            tb, te = C.c_int(0), C.c_int(self.plan.T)
            check(load().fqfg_das_slab_samples(self.plan.handle, kb, ke, C.byref(tb),
                                               C.byref(te)))
            hi = max(hi, min(te.value, self.t_end))
            lead.append((kb, ke, self.t_begin, hi))
        if lead:
            kb, ke, lo, _ = lead[-1]
            lead[-1] = (kb, ke, lo, self.t_end)
        self._lead = lead
        return lead

    def _lead_das(self, d_rf, xptr, cur, lead, wait):
        """Demod + DAS of the first streamed ensemble, sub-slab by sub-slab on
        torch stream `cur` (wait(i, stream) makes `stream` wait for sub-slab
        i's rows).  Single-pass plans demodulate incrementally
        (fqfg_das_dev_rows): sub-slab i makes the IQ rows whose FIR support its
        uploaded samples complete, so every row is demodulated once, as in one
        fqfg_das_dev call.  The demodulations run in order on `cur`; each
        sub-slab's DAS runs on its own stream after the demodulation that
        completes its rows (the rows a later demodulation writes and the voxels
        a later DAS writes are disjoint from what it reads and writes), so the
        next launch fills the SMs the previous one's tail frees; `cur` joins
        them all at the end."""
        torch = self.torch
        L = load()
        incremental = self.plan.n_passes == 1 and len(lead) > 1
        if not incremental:
            for i, (kb, ke, _, _) in enumerate(lead):
                wait(i, cur)
                self.plan.run(d_rf.data_ptr(), kb, ke, xptr, self.work.data_ptr(), None,
                              cur.cuda_stream)
            return
        if len(getattr(self, "_lead_streams", [])) < len(lead):
            self._lead_streams = [torch.cuda.Stream(self.device) for _ in range(len(lead))]
            self._lead_ev = [torch.cuda.Event() for _ in range(len(lead))]
        mid = self.plan.bp.lowpass_taps // 2
        T = self.plan.T
        # last IQ row made (row r = sample r - 1; rows 0 and T + 1 are guards):
        # a depth-slab rank holds RF [t_begin, t_end) only and reads IQ rows
        # (t_begin + mid, t_end - mid] (fqfg_das_slab_samples)
        done = self.t_begin + mid if self.t_begin > 0 else -1
        h, ptr, wk = self.plan.handle, d_rf.data_ptr(), self.work.data_ptr()
        for i, (kb, ke, _, hi) in enumerate(lead):
            # demodulation on `cur` (in order: sub-slab i's DAS reads rows
            # every earlier demodulation made), the DAS on its own stream
            wait(i, cur)
            last = T + 1 if hi >= T else hi - mid
            check(L.fqfg_das_dev_rows(h, ptr, kb, kb, done + 1, last, xptr, wk, None,
                                      cur.cuda_stream))
            done = max(done, last)
            ev, st = self._lead_ev[i], self._lead_streams[i]
            ev.record(cur)
            st.wait_event(ev)
            check(L.fqfg_das_dev_rows(h, ptr, kb, ke, 1, 0, xptr, wk, None, st.cuda_stream))
        for st in self._lead_streams[:len(lead)]:
            cur.wait_stream(st)

    def _run(self, inputs, host_pd, cur, before_step=None, after_das=None, first_das=None):
        """Reconstruct the ensembles inputs[k] (device RF tensors, or callables
        returning one after enqueuing its upload) with the cross-ensemble
        overlap; PD of ensemble k -> host_pd[k] (pinned; rank 0 when sharded)
        if given.  Sharded, the Gram all-reduce and the PD gather run on the
        filter stream too (every rank issues them in the same order), so the
        replicated eigensolve and the collectives overlap the next DAS."""
        torch = self.torch
        L = load()
        sharded = self.group is not None and self.world > 1
        if sharded:
            import torch.distributed as dist
        self._overlap_state()
        post = self._post
        post.wait_stream(cur)
        for k in range(len(inputs)):
            b = k % 2
            d_rf = inputs[k]() if callable(inputs[k]) else inputs[k]
            cur.wait_event(self._post_done[b])  # X[b] no longer read by ensemble k - 2
            s = cur.cuda_stream
            if k == 0 and first_das is not None:
                first_das(d_rf, self._xb[b].data_ptr(), s)
            else:
                self.plan.run(d_rf.data_ptr(), self.k0, self.k1, self._xb[b].data_ptr(),
                              self.work.data_ptr(), None, s)
            if after_das is not None:
                after_das(k)
            self._das_done[b].record(cur)
            post.wait_event(self._das_done[b])
            ps = post.cuda_stream
            check(L.fqfg_gram_dev(self._xb[b].data_ptr(), self.F, self.N, self.v0, self.v1,
                                  self._gb[b].data_ptr(), self._gwork.data_ptr(), ps))
            if sharded:
                with torch.cuda.stream(post):
                    dist.all_reduce(self._gb[b], group=self.group)
            check(L.fqfg_eig_band_dev(self._gb[b].data_ptr(), self.F, self.lo, self.hi,
                                      self._wb[b].data_ptr(), self._vb[b].data_ptr(), ps))
            check(L.fqfg_project_pd_dev(self._xb[b].data_ptr(), self.F, self.N, self.v0, self.v1,
                                        self._vb[b].data_ptr(), self.lo, self.hi, None,
                                        self._pdb[b].data_ptr(), ps))
            pd = self._pdb[b]
            if sharded:
                with torch.cuda.stream(post):
                    pd = gather_slabs(self._pdb[b], self.slabs, self.plan.grid.dims[0] *
                                      self.plan.grid.dims[1], self.group)
            if host_pd is not None and pd is not None:
                with torch.cuda.stream(post):
                    host_pd[k].copy_(pd, non_blocking=True)
            self._last_pd = pd
            self._post_done[b].record(post)
        cur.wait_stream(post)

    def run_resident(self, d_rf, steps, stream=None):
        """`steps` reconstructions of the device-resident RF d_rf (the bench's
        device-timed loop) with the cross-ensemble overlap (also when sharded:
        ensemble k's Gram all-reduce, eigensolve, projection and PD gather run
        on the filter stream during ensemble k+1's DAS).  Returns the last
        ensemble's PD (gathered on rank 0 when sharded, None elsewhere) and
        singular values."""
        torch = self.torch
        cur = torch.cuda.current_stream(self.device) if stream is None else stream
        self._run([d_rf] * steps, None, cur)
        return StepResult(self._last_pd,
                          torch.sqrt(torch.clamp(self._wb[(steps - 1) % 2], min=0.0)))

    def run_pipelined(self, host_rf, host_pd, stream=None):
        """Enqueue RF -> PD for a sequence of ensembles from pinned host memory:
        host_rf[k] ([F][A][T][E] f32, pinned) -> host_pd[k] ([N] f64, pinned;
        on rank 0 when sharded).  Two device input buffers and a copy stream:
        the upload of ensemble k+1 overlaps the reconstruction of ensemble k
        (and, on one GPU, ensemble k's filter overlaps ensemble k+1's DAS).
        Asynchronous; synchronise the stream before reading host_pd.  Returns
        the H2D bytes enqueued."""
        torch = self.torch
        if not hasattr(self, "_bufs"):
            self._bufs = [torch.empty(tuple(host_rf[0].shape), dtype=torch.float32,
                                      device=self.device) for _ in range(2)]
            self._copy = torch.cuda.Stream(self.device)
            self._copied = [torch.cuda.Event() for _ in range(2)]
            self._used = [torch.cuda.Event() for _ in range(2)]
            for e in self._used:
                e.record(torch.cuda.current_stream(self.device))
        cur = torch.cuda.current_stream(self.device) if stream is None else stream
        self._copy.wait_stream(cur)
        nbytes = [0]

        def upload(k):
            b = k % 2
            self._copy.wait_event(self._used[b])
            nbytes[0] += self.upload_rf(host_rf[k], self._bufs[b], self._copy.cuda_stream)
            self._copied[b].record(self._copy)

        # The first ensemble's upload is the only one nothing can hide: it
        # goes up in depth sub-slabs (rows each needs), and each sub-slab's
        # demod + DAS starts as soon as its rows are in.
        lead = self._lead_slabs() if len(host_rf) else []
        ev_lead = [torch.cuda.Event() for _ in lead]
        if lead:
            self._copy.wait_event(self._used[0])
            F, A, T, E = host_rf[0].shape
            row = E * 4
            lo = lead[0][2]
            for i, (_, _, _, hi) in enumerate(lead):
                if hi > lo:
                    check(load().fqfg_copy_slices_h2d(
                        self._bufs[0].data_ptr(), host_rf[0].data_ptr(), F * A, T * row,
                        lo * row, (hi - lo) * row, self._copy.cuda_stream))
                    nbytes[0] += F * A * (hi - lo) * row
                    lo = hi
                ev_lead[i].record(self._copy)
            self._copied[0].record(self._copy)

        def first_das(d_rf, xptr, s):
            self._lead_das(d_rf, xptr, cur, lead, lambda i, st: st.wait_event(ev_lead[i]))

        def source(k):
            def get():
                if k == 0 and not lead:
                    upload(0)
                if k + 1 < len(host_rf):
                    upload(k + 1)
                if k > 0 or not lead:
                    cur.wait_event(self._copied[k % 2])
                return self._bufs[k % 2]
            return get

        self._run([source(k) for k in range(len(host_rf))], host_pd, cur,
                  after_das=lambda k: self._used[k % 2].record(cur),
                  first_das=first_das if lead else None)
        return nbytes[0]

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
