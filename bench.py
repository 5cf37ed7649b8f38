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

value      whole-job nominal samples / s with RF already in HBM (device-timed,
           CUDA events on the working stream, max over ranks).
e2e        the same metric through the same public entry with RF copied
           host(pinned) -> device and PD device -> host inside every step.
roofline   the DAS kernel: 16 B per active (voxel, element, angle, frame)
           sample (two complex64 taps) / DAS kernel time.
cpu_baseline  the reference's own das_reconstruct (oracle/_ref, compiled from
           /root/reference) on a bounded sample, all host cores (rank 0, N=1).
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
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(self.rows)}
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
    sub = P.GridSpec((nx, ny, 1), g.spacing, (g.origin[0], g.origin[1],
                                               g.origin[2] + k * g.spacing[2]))
    F = 24
    rng = np.random.default_rng(1)
    rf = rng.uniform(-1, 1, (F, w.n_angles, w.n_samples, w.n_elements))
    rf = rf.astype(np.float32).astype(np.float64)
    return sub, rf


def run_cpu_reference(w, sub, rf):
    """The reference das_reconstruct (default DasOptions) + the FP64 filter
    restatement + power_doppler on the sample; returns (seconds, kind)."""
    from oracle import oracle as O
    os.environ.setdefault("FQF_THREADS", str(os.cpu_count()))
    t = time.perf_counter()
    if O.ref_available():
        iq, _ = O.ref_das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                          fc=w.fc)
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
            f"(plane {w.grid.dims[2] // 2} of {w.grid.dims[2]}), default DasOptions, "
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
        run_cpu_reference(w, sub, rf)
    times, kind = [], None
    for _ in range(args.steps):
        dt, kind = run_cpu_reference(w, sub, rf)
        times.append(dt)
    ms = 1000 * sum(times) / len(times)
    value = samples / (ms / 1000)
    cores = int(os.environ.get("FQF_THREADS", os.cpu_count()))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(w.describe(), sample=sample_desc(w, sub, rf)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample_desc(w, sub, rf)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours --

def ours(args):
    import torch
    import torch.distributed as dist

    import paper_2509_05464_b200 as P
    from paper_2509_05464_b200 import _native as N
    from paper_2509_05464_b200 import pipeline as PL
    from paper_2509_05464_b200 import workloads as W

    rank, world, local = dist_env()
    # FQFG_BENCH_DEVICE / FQFG_BENCH_BACKEND: functional checks of the N > 1
    # code path with several ranks on one GPU over gloo (not a measurement).
    if os.environ.get("FQFG_BENCH_DEVICE") is not None:
        local = int(os.environ["FQFG_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    # Config E (batch sweep of ensembles): every GPU reconstructs whole
    # ensembles of its own (replicas, no data-path collective); otherwise the
    # ensemble is depth-slab sharded over the ranks.
    replicas = args.config.upper() == "E"
    if world > 1:
        backend = os.environ.get("FQFG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        if not replicas:
            group = dist.group.WORLD
    L = N.load()
    w = W.config(args.config)
    F, A, T, E = w.rf_shape()
    rec = PL.Reconstructor(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), keep_lo=2,
                           keep_hi=F, group=group, device=dev)
    stream = torch.cuda.current_stream(dev)
    d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device=dev)
    N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 20260816 + (rank if replicas else 0),
                                stream.cuda_stream))
    pairs = PL.active_pairs_per_plane(w.grid, w.elements, w.bf().f_number)
    active_rank = float(pairs[rec.k0:rec.k1].sum()) * A * F  # active samples of this rank

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # Steps run back to back through Reconstructor.run_resident: on one GPU
    # ensemble k's filter (Gram, one-CTA eigensolve, projection) overlaps
    # ensemble k+1's demod + DAS on a second stream.
    rec.run_resident(d_rf, args.warmup)
    torch.cuda.synchronize()

    # ---- device-resident timed region
    L.fqfg_das_plan_set_timing(rec.plan.handle, 1)
    launches0 = L.fqfg_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        out = rec.run_resident(d_rf, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    barrier()
    launches = L.fqfg_launch_count() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    dm, da = __import__("ctypes").c_double(), __import__("ctypes").c_double()
    N.check(L.fqfg_das_last_timing(rec.plan.handle, dm, da))
    L.fqfg_das_plan_set_timing(rec.plan.handle, 0)
    das_ms = da.value / args.steps
    demod_ms = dm.value / args.steps
    das_ms_max = max_over_ranks(das_ms)
    clocks = clk.summary()

    # ---- end to end: pinned host RF in, PD out, inside every step
    e2e = None
    if not args.no_e2e:
        h_rf = torch.empty(w.rf_shape(), dtype=torch.float32, pin_memory=True)
        h_rf.copy_(d_rf)
        h_pd = torch.empty(w.grid.num_points(), dtype=torch.float64, pin_memory=True)
        # Streaming: the upload of ensemble k+1 (copy stream, only the RF
        # samples this rank's slab reads) overlaps the reconstruction of k;
        # every step's H2D copy and PD read-back are inside the timed region.
        rec.run_pipelined([h_rf], [h_pd])
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        rec.run_pipelined([h_rf] * args.steps, [h_pd] * args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        h2d_rank = F * A * (rec.t_end - rec.t_begin) * E * 4
        h2d = h2d_rank
        if world > 1:
            t = torch.tensor([float(h2d_rank)], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            h2d = int(t.item())
        d2h = h_pd.numel() * 8
        e2e = {"value": w.nominal_samples() * (world if replicas else 1) / (e2e_ms / 1000),
               "unit": UNIT,
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pd_volumes_per_s": 1000.0 / e2e_ms,
               "entry": "paper_2509_05464_b200.pipeline.Reconstructor.run_pipelined "
                        "(pinned host RF -> host PD, upload of k+1 overlapping step k)"}

    # ---- the filter stages timed one by one (after the timed region): Gram
    # (FP64, 8 N F^2 useful flops; the SURVEY 8(d) filter roofline), the
    # eigensolve and the projection + PD (2 passes over X: 16 N F bytes).
    filt = None
    try:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ss = stream.cuda_stream
        nrep = 3
        ev[0].record(stream)
        for _ in range(nrep):
            N.check(L.fqfg_gram_dev(rec.x.data_ptr(), F, rec.N, rec.v0, rec.v1, rec.gram.data_ptr(),
                                    rec.work.data_ptr(), ss))
        ev[1].record(stream)
        g_copy = rec.gram.clone()
        for _ in range(nrep):
            rec.gram.copy_(g_copy)
            N.check(L.fqfg_eig_band_dev(rec.gram.data_ptr(), F, rec.lo, rec.hi, rec.w.data_ptr(),
                                        rec.v.data_ptr(), ss))
        ev[2].record(stream)
        for _ in range(nrep):
            N.check(L.fqfg_project_pd_dev(rec.x.data_ptr(), F, rec.N, rec.v0, rec.v1,
                                          rec.v.data_ptr(), 2, F, None, rec.pd.data_ptr(), ss))
        ev[3].record(stream)
        torch.cuda.synchronize()
        gram_ms = ev[0].elapsed_time(ev[1]) / nrep
        eig_ms = ev[1].elapsed_time(ev[2]) / nrep - 0.0
        proj_ms = ev[2].elapsed_time(ev[3]) / nrep
        nvox = rec.v1 - rec.v0
        # algorithmic flops: the Hermitian upper triangle (F (F + 1) / 2 complex
        # multiply-adds of 8 flops per voxel); the kernel also computes the
        # padding / lower half of its diagonal tiles (see "executed_flops")
        gram_tf = 8.0 * nvox * F * (F + 1) / 2 / (gram_ms / 1e3) / 1e12
        tb, cost = None, None  # the FP64 tile choice of gram_tile (csrc/capi.cu)
        for t in (64, 48, 40, 32):
            nb = -(-F // t)
            c = nb * (nb + 1) // 2 * t * t
            if cost is None or c < cost:
                cost, tb = c, t
        dfma_peak = 35.6
        try:
            hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            hbm_peak = 6650.0
        filt = {"gram_ms": gram_ms, "eig_ms": eig_ms, "project_pd_ms": proj_ms,
                "gram": {"bound": "fp64", "achieved": gram_tf, "peak": dfma_peak,
                         "unit": "TFLOP/s", "frac": gram_tf / dfma_peak,
                         "flops": "8 x voxels x F (F + 1) / 2 (upper triangle)",
                         "tile": tb, "executed_flops": 8.0 * nvox * cost,
                         "executed_tflops": 8.0 * nvox * cost / (gram_ms / 1e3) / 1e12,
                         "peak_source": "measured DFMA throughput on B200 (scripts/microbench/"
                                        "fp64_bench.cu); FP64 tensor cores (mma.sync f64) "
                                        "measure 37.2"},
                # default band [2, F]: rank-1 complement, one streaming pass over
                # X (8 N F bytes) plus the f64 PD write
                "project_pd": {"bound": "hbm",
                               "achieved": (8.0 * nvox * F + 8.0 * nvox) / (proj_ms / 1e3) / 1e9,
                               "peak": hbm_peak, "unit": "GB/s",
                               "frac": (8.0 * nvox * F + 8.0 * nvox) / (proj_ms / 1e3) / 1e9
                               / hbm_peak}}
    except Exception as ex:  # reporting only
        filt = {"error": str(ex)}

    # ---- roofline of the dominant kernel (DAS)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, peak_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        hbm, peak_src = 6650.0, "fallback"
    active_total = max_over_ranks(active_rank) if world > 1 else active_rank
    achieved = 16.0 * active_rank / (das_ms / 1000) / 1e9 if das_ms > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "das_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config.upper())
        except Exception:
            traffic = None
    # The taps are served from shared memory (traffic << algorithmic bytes), so
    # the binding resource is shared-memory bandwidth: 128 B/clk/SM x 148 SMs
    # at the SM clock measured during the timed region.
    sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
    smem_peak = 148 * 128 * sm_hz / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                "kernel": "das2_kernel (mode 0; frames/pass %d, voxel tile %s)" % (
                         rec.plan.frames_per_pass, "x".join(map(str, rec.plan.tile))),
                "binding_resource": {"name": "shared-memory bandwidth (128 B/clk/SM)",
                                     "peak_GBs": smem_peak,
                                     "frac": (achieved / smem_peak) if achieved else None},
                "peak_source": peak_src + " MEASURED_PEAKS.json hbm_gbs",
                "unit_bytes": "16 B per active voxel-element-angle-frame sample (SURVEY 8(d))",
                "das_ms_per_step": das_ms, "demod_ms_per_step": demod_ms,
                "active_fraction": float(pairs.sum()) / (w.grid.num_points() * E)}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sub, rf = cpu_sample(w)
            dt, kind = run_cpu_reference(w, sub, rf)
            samples = sub.num_points() * w.n_elements * w.n_angles * rf.shape[0]
            cpu = {"value": samples / dt, "unit": UNIT,
                   "cores": int(os.environ.get("FQF_THREADS", os.cpu_count())), "kind": kind,
                   "sample": sample_desc(w, sub, rf), "seconds": dt}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {ex}"}

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
                               l2="inputs larger than L2 (RF %.1f GB per step)"
                               % (d_rf.numel() * 4 / 1e9),
                               precision="f32 IQ/gather/accumulate, f64 delays, Gram, eig, PD"),
                "pd_volumes_per_s": 1000.0 * (world if replicas else 1) / ms,
                "stages_ms": {"demod": demod_ms, "das": das_ms, "das_max_rank": das_ms_max,
                              "filter_and_rest_not_overlapped": ms - demod_ms - das_ms},
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
                "gpu_launches": int(launches), "filter_roofline": filt}
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
