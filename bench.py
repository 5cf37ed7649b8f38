#!/usr/bin/env python
"""Benchmark: RF channel data -> IQ demod -> 3D plane-wave DAS -> Casorati SVD
clutter filter -> power Doppler, one ensemble per step (BASELINE.json metric:
beamformed voxel x element x angle samples/s, plus PD volumes/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

N > 1: launched under torch.distributed.run, one rank per GPU, NCCL; the
ensemble is depth-slab sharded (the per-slab Gram is the only collective), so
total work is fixed: "scaling": "strong".  --config E (the batch sweep) runs
ensemble replicas instead: each GPU reconstructs its own ensemble per step, no
collective, "scaling": "weak".  Rank 0 prints one JSON line.

Both arms of ours go through the C ABI of the C++ reconstruction engine
(fqfg_recon_*, csrc/recon.cu):
value      whole-job nominal samples / s with RF already in HBM
           (fqfg_recon_run_dev; device time of the whole run from CUDA events
           on the engine's streams, max over ranks).
e2e        the same metric through fqfg_recon_run with RF in pinned host
           memory: every step's RF upload and PD read-back inside the timing.
roofline   the DAS kernel: 16 B per active (voxel, element, angle, frame)
           sample (two complex64 taps) / DAS kernel time,
           against its binding resource (measured shared-memory bandwidth);
           the SURVEY's HBM-normalised figure is kept under hbm_normalised.
filter_roofline  Gram + eigensolve + projection vs SURVEY 8(d)'s tensor roofline.
cpu_baseline  the reference's own das_reconstruct (oracle/_ref, compiled from
           /root/reference) on a bounded sample, all host cores (rank 0, N=1).
parity     the benchmarked run's own IQ / PD on a voxel block vs the reference
           (checker only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "beamformed voxel-element-angle samples/s"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C",
                    help="workload A-E (BASELINE.json configs); E = ensemble replicas of C")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a moment to start: the timed region begins only
            # once it is sampling.
            t = time.time()
            while not self.rows and time.time() - t < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        self.first = len(self.rows)
        return self

    def mark_end(self):
        """End of the timed region; a region shorter than the sampling period
        gets the first sample after it."""
        self.last = len(self.rows)
        if self.proc and self.last == self.first:
            t = time.time()
            while len(self.rows) == self.last and time.time() - t < 1.0:
                time.sleep(0.01)
            self.after = True
        else:
            self.after = False

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        last = getattr(self, "last", len(self.rows))
        rows = self.rows[self.first:max(last, self.first + 1)] if getattr(self, "after", False) \
            else self.rows[self.first:last] or self.rows[-1:]
        self.rows = rows
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v == "Active"})
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[3]))
            except ValueError:
                pass
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(self.rows),
               "power_w": statistics.median(pw) if pw else None}
        if getattr(self, "after", False):
            out["note"] = "timed region shorter than the 100 ms sampling period: first sample after it"
        return out


# ------------------------------------------------------------- CPU sample --

def cpu_sample(w, budget_s=None):
    """A bounded slice of the workload for the CPU reference (about 10 s of
    16-core work at config C): 24 frames, all angles and elements, the full
    lateral plane of voxels at mid depth."""
    import paper_2509_05464_b200 as P
    g = w.grid
    nx, ny, nz = g.dims
    k = nz // 2
    # the reference builds each chunk's delay matrices serially (~1.4e7
    # voxel-element pairs / s): keep voxels x elements x angles near 1.5e8
    bx, by = nx, ny
    while bx * by * w.n_elements * w.n_angles > 1.6e8 and bx > 8:
        bx, by = bx // 2, max(by // 2, 1)
    sub = P.GridSpec((bx, by, 1), g.spacing,
                     (g.origin[0] + (nx - bx) // 2 * g.spacing[0],
                      g.origin[1] + (ny - by) // 2 * g.spacing[1], g.origin[2] + k * g.spacing[2]))
    F = 24 if w.n_elements * w.n_samples <= 1024 * 1024 else 8
    rng = np.random.default_rng(1)
    rf = rng.uniform(-1, 1, (F, w.n_angles, w.n_samples, w.n_elements))
    rf = rf.astype(np.float32).astype(np.float64)
    return sub, rf


def host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 64 << 30


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_cpu_reference(w, sub, rf, tuned=False):
    """The reference das_reconstruct + the FP64 filter restatement +
    power_doppler on the sample; returns (seconds, kind).  tuned: the
    matrix budget raised to half the host RAM (SURVEY 8(d) "tuned": one chunk,
    no repeated demodulation), else the default DasOptions (das.hpp:101-108)."""
    from oracle import oracle as O
    os.environ.setdefault("FQF_THREADS", str(os.cpu_count()))
    kw = dict(matrix_budget=host_ram_bytes() // 2, memory_budget=host_ram_bytes() // 8) \
        if tuned else {}
    t = time.perf_counter()
    if O.ref_available():
        iq, _ = O.ref_das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                          fc=w.fc, **kw)
        kind = "reference"
    else:
        iq, _ = O.das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                      fc=w.fc)
        kind = "port"
    y, _, _ = O.svd_filter(iq, 2, iq.shape[0], method="gram")
    O.power_doppler(y)
    return time.perf_counter() - t, kind


def sample_desc(w, sub, rf):
    return (f"{w.name.split(':')[0]} geometry, {rf.shape[0]} frames x {w.n_angles} angles x "
            f"{w.n_elements} elements x {sub.dims[0]}x{sub.dims[1]}x{sub.dims[2]} voxels "
            f"(plane {w.grid.dims[2] // 2} of {w.grid.dims[2]}), reference das_reconstruct, "
            f"+ FP64 SVD-filter restatement + power_doppler")


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2509_05464_b200 import workloads as W
    w = W.config(args.config)
    sub, rf = cpu_sample(w)
    samples = sub.num_points() * w.n_elements * w.n_angles * rf.shape[0]
    for _ in range(args.warmup):
        run_cpu_reference(w, sub, rf, tuned=True)
    times, kind = [], None
    for _ in range(args.steps):
        dt, kind = run_cpu_reference(w, sub, rf, tuned=True)
        times.append(dt)
    ms = 1000 * sum(times) / len(times)
    value = samples / (ms / 1000)
    dt_default, _ = run_cpu_reference(w, sub, rf, tuned=False)
    cores = int(os.environ.get("FQF_THREADS", os.cpu_count()))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(w.describe(), sample=sample_desc(w, sub, rf)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample_desc(w, sub, rf) + "; matrix budget = half the "
                                       "host RAM (tuned)", "cpu_model": cpu_model(),
                             "default_das_options": {"value": samples / dt_default,
                                                     "seconds": dt_default}},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours --

def parity_leg(w, eng, d_rf, kb):
    """Parity of the benchmarked run itself (rank 0, N = 1): the IQ the
    production engine made for an 8 x 8 x 4 voxel block at mid depth of the
    full grid (its last timed ensemble, same RF) against the reference's own
    das_reconstruct (oracle/_ref) on that block; and the PD of the same block
    reconstructed by the engine at the full frame count (F = 200 at C: the
    production kernel shapes and filter) against the FP64 SVD-filter
    restatement + power_doppler of the reference IQ.  Checker only: the
    oracle never runs on the product path."""
    import torch
    import paper_2509_05464_b200 as P
    from oracle import oracle as O
    from paper_2509_05464_b200.engine import Engine
    g = w.grid
    nx, ny, nz = g.dims
    bx, by = 8 if ny > 1 else 16, min(8, ny)
    bz = max(4, -(-w.n_frames // (bx * by)))  # svd_filter needs F <= voxels
    i0, j0 = nx // 2 - bx // 2, max(ny // 2 - by // 2, 0)
    k0 = kb if kb is not None else nz // 2
    if ny == 1:
        # config A's lattice (lambda/2 voxels, 0.3 mm pitch) puts many voxels
        # exactly on the f-number boundary, where origin + i * spacing of a
        # sub-grid and of the full grid round differently; at the grid's own
        # origin the block's coordinates are the full grid's, bit for bit
        i0 = k0 = 0
    sub = P.GridSpec((bx, by, bz), g.spacing,
                     tuple(g.origin[d] + (i0, j0, k0)[d] * g.spacing[d] for d in range(3)))
    rf = d_rf.cpu().numpy()
    t = time.perf_counter()
    iq_ref, _ = O.ref_das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                          fc=w.fc)
    ref_s = time.perf_counter() - t
    plane = nx * ny
    full = eng.copy_iq(k0 * plane, (k0 + bz) * plane).reshape(w.n_frames, bz, ny, nx)
    iq_gpu = full[:, :, j0:j0 + by, i0:i0 + bx].reshape(w.n_frames, -1)
    e_iq = float(np.linalg.norm(iq_gpu - iq_ref) / np.linalg.norm(iq_ref))
    sub_eng = Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, sub, w.elements, w.bf())
    pd = np.zeros(sub.num_points())
    sub_eng.run([rf], [pd])
    iq_sub = sub_eng.copy_iq()
    shape = tuple(sub_eng.info.shape)
    sub_eng.close()
    y, _, _ = O.svd_filter(iq_ref, 2, w.n_frames, method="gram")
    pd_ref = O.power_doppler(y)
    e_pd = float(np.linalg.norm(pd - pd_ref) / np.linalg.norm(pd_ref))
    e_iq_sub = float(np.linalg.norm(iq_sub - iq_ref) / np.linalg.norm(iq_ref))
    return {"iq_rel_l2": e_iq, "pd_rel_l2": e_pd, "iq_rel_l2_block_engine": e_iq_sub,
            "tolerance": {"iq_rel_l2": 1e-5, "pd_rel_l2": 1e-4},
            "pass": e_iq < 1e-5 and e_pd < 1e-4 and e_iq_sub < 1e-5,
            "sample": f"voxel block {bx}x{by}x{bz} at grid index ({i0}, {j0}, {k0}), all "
                      f"{w.n_elements} elements x {w.n_angles} angles x {w.n_frames} frames of "
                      f"the bench's own synthetic RF; IQ from the full-grid timed run; PD from "
                      f"the engine on the block (kernel shape J,VPW,NW,PW = {shape}) vs the "
                      f"reference das_reconstruct + FP64 filter restatement + power_doppler",
            "reference_seconds": ref_s}


def filter_standalone(L, N, F, nloc, dev, nrep=3):
    """Gram (the engine's tensor-core kernel), band eigensolve and projection
    + PD timed one by one on a synthetic X of the slab's shape (in the
    pipeline they overlap the next DAS, so their span there is not their
    cost)."""
    import torch
    x = torch.randn((F, max(nloc, 1), 2), dtype=torch.float32, device=dev)
    gram = torch.empty((F, F, 2), dtype=torch.float64, device=dev)
    g2 = torch.empty_like(gram)
    wv = torch.empty(F, dtype=torch.float64, device=dev)
    v = torch.empty_like(gram)
    pd = torch.empty(max(nloc, 1), dtype=torch.float64, device=dev)
    work = torch.empty(L.fqfg_gram_tc_work_bytes(F), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    ss = s.cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    N.check(L.fqfg_gram_tc_dev(x.data_ptr(), F, nloc, 0, nloc, gram.data_ptr(), work.data_ptr(),
                               ss))
    ev[0].record(s)
    for _ in range(nrep):
        N.check(L.fqfg_gram_tc_dev(x.data_ptr(), F, nloc, 0, nloc, gram.data_ptr(),
                                   work.data_ptr(), ss))
    ev[1].record(s)
    for _ in range(nrep):
        g2.copy_(gram)
        N.check(L.fqfg_eig_band_dev(g2.data_ptr(), F, 2, F, wv.data_ptr(), v.data_ptr(), ss))
    ev[2].record(s)
    for _ in range(nrep):
        N.check(L.fqfg_project_pd_dev(x.data_ptr(), F, nloc, 0, nloc, v.data_ptr(), 2, F, None,
                                      pd.data_ptr(), ss))
    ev[3].record(s)
    torch.cuda.synchronize(dev)
    return (ev[0].elapsed_time(ev[1]) / nrep, ev[1].elapsed_time(ev[2]) / nrep,
            ev[2].elapsed_time(ev[3]) / nrep)


def ours(args):
    import torch
    import torch.distributed as dist

    from paper_2509_05464_b200 import _native as N
    from paper_2509_05464_b200 import workloads as W
    from paper_2509_05464_b200.engine import Engine, nccl_unique_id

    rank, world, local = dist_env()
    # FQFG_BENCH_DEVICE / FQFG_BENCH_BACKEND: functional checks of the N > 1
    # code path with several ranks on one GPU over gloo (not a measurement).
    if os.environ.get("FQFG_BENCH_DEVICE") is not None:
        local = int(os.environ["FQFG_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # Config E (batch sweep of ensembles): every GPU reconstructs whole
    # ensembles of its own (replicas, no data-path collective); otherwise the
    # ensemble is depth-slab sharded over the ranks.
    replicas = args.config.upper() == "E"
    backend = os.environ.get("FQFG_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    sharded = world > 1 and not replicas
    L = N.load()
    w = W.config(args.config)
    F, A, T, E = w.rf_shape()
    kw = {}
    if sharded:
        if backend == "nccl":
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            kw = dict(rank=rank, world=world, nccl_id=obj[0])
        else:  # several ranks on one GPU: NCCL refuses that, sum the Gram over gloo
            import ctypes as C
            cudart = C.CDLL("libcudart.so")

            def allreduce(ptr, n, stream):
                buf = np.empty(n, np.float64)
                cudart.cudaStreamSynchronize(C.c_void_p(stream))
                cudart.cudaMemcpy(C.c_void_p(buf.ctypes.data), C.c_void_p(ptr), C.c_size_t(8 * n), 2)
                t = torch.from_numpy(buf)
                dist.all_reduce(t)
                return int(cudart.cudaMemcpy(C.c_void_p(ptr), C.c_void_p(buf.ctypes.data),
                                             C.c_size_t(8 * n), 1))
            kw = dict(rank=rank, world=world, allreduce=allreduce)
    eng = Engine(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), keep_lo=2, keep_hi=F, **kw)
    info = eng.info
    seed = 20260816 + (rank if replicas else 0)
    rf_bytes = 4 * F * A * T * E
    # Config D's RF (115 GB) cannot stay resident next to its IQ pass and X:
    # it is streamed from pinned host memory in every timed step, so `value`
    # and `e2e` are the same measurement there.
    streamed = rf_bytes > 0.25 * torch.cuda.get_device_properties(dev).total_memory
    d_rf, h_rf = None, None
    if streamed:
        h_rf = torch.empty(w.rf_shape(), dtype=torch.float32, pin_memory=True)
        scratch = torch.empty((16,) + w.rf_shape()[1:], dtype=torch.float32, device=dev)
        for f0 in range(0, F, 16):
            n = min(16, F - f0)
            N.check(L.fqfg_synth_rf_dev(scratch.data_ptr(), n * A * T * E, seed + f0,
                                        torch.cuda.current_stream(dev).cuda_stream))
            h_rf[f0:f0 + n].copy_(scratch[:n])
        del scratch
    else:
        d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device=dev)
        N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), seed,
                                    torch.cuda.current_stream(dev).cuda_stream))
    torch.cuda.synchronize(dev)
    h_pd = torch.empty(w.grid.num_points(), dtype=torch.float64, pin_memory=True)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t)
        return float(t.item())

    # ---- device-resident RF: steps back to back through the engine (the
    # filter of ensemble k overlaps the demod + DAS of k + 1).
    def timed_run(k):
        if streamed:
            eng.run([h_rf] * k, [h_pd] * k)
        else:
            eng.run_dev([d_rf] * k)

    timed_run(args.warmup)
    eng.set_timing(True)
    launches0 = L.fqfg_launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        timed_run(args.steps)
        wall = time.perf_counter() - wall0
        clk.mark_end()
    barrier()
    launches = L.fqfg_launch_count() - launches0
    demod_ms, das_ms, filt_span_ms, total_ms = eng.last_timing()
    kblocks = eng.mma_blocks() / args.steps  # tensor-core DAS K blocks per step (0: das2)
    ms = max_over_ranks(total_ms) / args.steps
    das_ms /= args.steps
    demod_ms /= args.steps
    das_ms_max = max_over_ranks(das_ms)
    clocks = clk.summary()

    # ---- end to end through the C ABI (fqfg_recon_run): pinned host RF in,
    # host PD out, every step's upload and read-back inside the timed region.
    e2e = None
    if not args.no_e2e:
        if streamed:  # the timed run above already streamed RF from the host
            e2e_wall, e2e_ms = wall, ms * args.steps
        else:
            h_rf = torch.empty(w.rf_shape(), dtype=torch.float32, pin_memory=True)
            h_rf.copy_(d_rf)
            eng.run([h_rf], [h_pd])
            barrier()
            wall0 = time.perf_counter()
            eng.run([h_rf] * args.steps, [h_pd] * args.steps)
            e2e_wall = time.perf_counter() - wall0
            barrier()
            e2e_ms = max_over_ranks(eng.last_timing()[3])
        e2e_ms /= args.steps
        h2d = sum_over_ranks(info.h2d_bytes_per_ensemble)
        d2h = h_pd.numel() * 8 if not sharded else sum_over_ranks((info.v_end - info.v_begin) * 8)
        e2e = {"value": w.nominal_samples() * (world if replicas else 1) / (e2e_ms / 1000),
               "unit": UNIT, "ms_per_step": e2e_ms, "wall_ms_per_step": 1000 * e2e_wall / args.steps,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "h2d_bytes_per_rank": int(info.h2d_bytes_per_ensemble),
               "pd_volumes_per_s": 1000.0 * (world if replicas else 1) / e2e_ms,
               "entry": "C ABI fqfg_recon_run (C++ engine, csrc/recon.cu): pinned host RF "
                        "-> host PD; RF uploaded 16 frames at a time into a staging ring "
                        "(only the samples the voxels can read) overlapping demod + DAS"}

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, peak_src = float(peaks["hbm_gbs"]), "measured MEASURED_PEAKS.json"
    except Exception:
        hbm, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    tensor_peak = float(peaks.get("bf16_tflops_sustained", 1388.8))
    nloc = int(info.v_end - info.v_begin)
    # ---- roofline of the dominant kernel (DAS): its taps come from shared
    # memory, so the binding resource is shared-memory bandwidth (measured
    # LDS peak, scripts/microbench/lds_bench.cu -> profiles/smem_peak.json).
    active_rank = float(info.active_samples)
    achieved = 16.0 * active_rank / (das_ms / 1000) / 1e9 if das_ms > 0 else None
    sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
    try:
        sp = json.load(open(os.path.join(ROOT, "profiles", "smem_peak.json")))
        bpc, smem_src = float(sp["bytes_per_clk_sm"]), sp["source"]
    except Exception:
        bpc, smem_src = 128.0, "nominal 128 B/clk/SM (no measurement file)"
    smem_peak = 148 * bpc * sm_hz / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "das_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config.upper())
        except Exception:
            traffic = None
    rows = info.t_end - info.t_begin
    compulsory = A * E * rows * 8.0 * info.frames_per_pass * info.n_passes + 8.0 * F * nloc
    useful = {"unit_flops": "16 flops per active voxel-element-angle-frame sample (two complex "
                            "taps x complex weight, SURVEY 8(d))",
              "useful_tflops": 16.0 * active_rank / (das_ms / 1000) / 1e12 if das_ms > 0 else None,
              "smem_normalised": {"achieved_gbs": achieved, "peak_gbs": smem_peak,
                                  "frac": (achieved / smem_peak) if achieved else None,
                                  "unit": "16 B per active sample (the das2 gather's bytes)",
                                  "peak_source": f"{bpc:.1f} B/clk/SM ({smem_src})"},
              "hbm_normalised": {"achieved": achieved, "peak": hbm,
                                 "frac": (achieved / hbm) if achieved else None,
                                 "peak_source": peak_src,
                                 "note": "SURVEY 8(d)'s effective-gather definition; above 1 "
                                         "because the taps never come from HBM one by one"}}
    if info.mode == 2:
        # das_tc_kernel: the binding resource is the tensor pipe.  Work per K
        # block = 3 tcgen05.mma kind::f16 (hi.hi, hi.lo, lo.hi) of M 128 x
        # N frames_per_pass x K 16; K blocks counted on the device.
        fl = kblocks * 3 * 2.0 * 128 * info.frames_per_pass * 16
        mma_tf = fl / (das_ms / 1000) / 1e12 if das_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": mma_tf, "peak": tensor_peak, "unit": "TFLOP/s",
                    "frac": (mma_tf / tensor_peak) if mma_tf else None, "traffic": traffic,
                    "kernel": "das_tc_kernel (tcgen05.mma kind::f16, A = weights in TMEM, B = "
                              "fp16 hi/lo IQ row chunks in shared memory), tile %s, %d frames/pass"
                              % ("x".join(map(str, info.tile)), info.frames_per_pass),
                    "peak_source": "dense f16/bf16 tensor peak, sustained (MEASURED_PEAKS.json "
                                   "bf16_tflops_sustained; kind::f16 runs at the bf16 rate)",
                    "unit_flops": "per K block 3 x 2 x 128 x frames_per_pass x 16 (the MMAs "
                                  "this formulation issues; counted live: %d K blocks per step)"
                                  % int(kblocks),
                    "mma_kblocks_per_step": kblocks, "useful": useful,
                    "compulsory_dram_bytes": compulsory,
                    "compulsory_note": "IQ windows read once + X written once per step",
                    "das_ms_per_step": das_ms, "demod_ms_per_step": demod_ms,
                    "active_samples": active_rank}
    else:
        roofline = {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                    "frac": (achieved / smem_peak) if achieved else None, "traffic": traffic,
                    "kernel": "das2_kernel<J=%d,VPW=%d,NW=%d,PW=%d>, tile %s, %d frames/pass" % (
                        tuple(info.shape) + ("x".join(map(str, info.tile)), info.frames_per_pass)),
                    "peak_source": f"{bpc:.1f} B/clk/SM ({smem_src}) x 148 SMs x median SM clock "
                                   f"under load",
                    "unit_bytes": "16 B per active voxel-element-angle-frame sample (two complex64 "
                                  "taps, SURVEY 8(d)), all served from shared memory",
                    "hbm_normalised": useful["hbm_normalised"],
                    "compulsory_dram_bytes": compulsory,
                    "compulsory_note": "IQ windows read once + X written once per step",
                    "das_ms_per_step": das_ms, "demod_ms_per_step": demod_ms,
                    "active_samples": active_rank}

    # ---- CPU baseline + parity of this run (rank 0, N = 1 only)
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sub, rf = cpu_sample(w)
            dt, kind = run_cpu_reference(w, sub, rf, tuned=True)
            samples = sub.num_points() * w.n_elements * w.n_angles * rf.shape[0]
            cpu = {"value": samples / dt, "unit": UNIT,
                   "cores": int(os.environ.get("FQF_THREADS", os.cpu_count())), "kind": kind,
                   "sample": sample_desc(w, sub, rf) + "; matrix budget = half the host RAM "
                                                       "(tuned)",
                   "seconds": dt, "cpu_model": cpu_model()}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {ex}"}
        if streamed:
            parity = {"skipped": "the reference das_reconstruct needs the whole RF in FP64 "
                                 "(%.0f GB) on the host; config-D geometry parity is covered by "
                                 "tests/test_gpu_parity.py::test_das_at_config_d_geometry"
                                 % (2 * rf_bytes / 1e9)}
        elif not args.no_parity:
            try:
                parity = parity_leg(w, eng, d_rf, None)
            except Exception as ex:
                parity = {"error": str(ex)}

    # ---- the filter stages standalone (SURVEY 8(d) tensor roofline: 8 N F^2
    # useful flops for the Gram + 8 N F^2 for the projection, 16 N F + 4 N bytes)
    # (run after the engine released its buffers: at config D it holds ~146 GB)
    eng.close()
    del d_rf
    torch.cuda.empty_cache()
    try:
        gram_ms, eig_ms, proj_ms = filter_standalone(L, N, F, nloc, dev)
    except Exception as ex:  # reporting only
        gram_ms = eig_ms = proj_ms = None
        filt = {"error": str(ex)}
    if gram_ms is not None:
        fl = 16.0 * nloc * F * F
        by = 16.0 * nloc * F + 4.0 * nloc
        t_roof = max(fl / (tensor_peak * 1e12), by / (hbm * 1e9)) * 1e3
        t_meas = gram_ms + eig_ms + proj_ms
        filt = {"bound": "tensor", "gram_ms": gram_ms, "eig_ms": eig_ms, "project_pd_ms": proj_ms,
                "roofline_ms": t_roof, "frac": t_roof / t_meas,
                "useful_tflops": fl / (t_meas * 1e-3) / 1e12, "peak_tflops": tensor_peak,
                "definition": "SURVEY 8(d): max(16 N F^2 flops / bf16 sustained, (16 N F + 4 N) B "
                              "/ HBM) over the measured Gram + eigensolve + projection time",
                "gram_engine": "tensor cores: tcgen05.mma kind::i8 on 4 x 7-bit digit planes per "
                               "sample, int32 TMEM accumulation, FP64 recombination "
                               "(csrc/gram_i8.cu; ~1e-10 of the largest entry vs exact FP64)",
                "span_in_pipeline_ms": filt_span_ms / args.steps}

    if rank == 0:
        # whole-job throughput: with replicas every rank finished its own ensemble
        value = w.nominal_samples() * (world if replicas else 1) / (ms / 1000)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak" if replicas else "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(w.describe(),
                               parallelism=(f"ensemble replicas x{world} (one ensemble per GPU "
                                            "per step)" if replicas else
                                            f"depth-slab x{world}" if world > 1
                                            else "single GPU"), band=[2, F],
                               l2="inputs larger than L2 (RF %.1f GB per step)" % (rf_bytes / 1e9),
                               rf=("streamed from pinned host memory every step (does not fit "
                                   "HBM next to the IQ pass and X): value = e2e" if streamed
                                   else "resident in HBM for value, pinned host memory for e2e"),
                               precision=("DAS on tensor cores: IQ and weights split fp16 "
                                          "hi + lo (products ~2^-22 relative), fp32 "
                                          "accumulation restarted every 16 stages; f64 "
                                          "delays, Gram (int8 digits, FP64 sums), eig, PD"
                                          if info.mode == 2 else
                                          "f32 IQ/gather/accumulate, f64 delays, Gram, eig, "
                                          "PD")),
                "entry": ("C ABI fqfg_recon_run (C++ engine): RF streamed from pinned host "
                          "memory" if streamed else
                          "C ABI fqfg_recon_run_dev (C++ engine): device-resident RF") +
                         " -> PD, device time of the whole run (CUDA events), max over ranks",
                "wall_ms_per_step": 1000 * wall / args.steps,
                "pd_volumes_per_s": 1000.0 * (world if replicas else 1) / ms,
                "stages_ms": {"demod": demod_ms, "das": das_ms, "das_max_rank": das_ms_max,
                              "filter_span_overlapped": filt_span_ms / args.steps},
                "engine": {"frames_per_pass": info.frames_per_pass, "passes": info.n_passes,
                           "x_buffers": info.x_buffers, "ring_frames": info.ring_frames,
                           "device_gb": info.device_bytes / 1e9, "rf_window": [info.t_begin,
                                                                               info.t_end],
                           "slab_planes": [info.k_begin, info.k_end], "nccl": bool(info.nccl)},
                "e2e": e2e, "roofline": roofline, "filter_roofline": filt,
                "cpu_baseline": cpu, "parity": parity, "clocks": clocks,
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


if __name__ == "__main__":
    sys.exit(main())
