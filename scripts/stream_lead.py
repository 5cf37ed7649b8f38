"""Times the first-ensemble streaming variants (profiles/r01_stream_lead.md): e2e
run_pipelined at K = 1 and 5 for several sub-slab cuts.  Usage: python scripts/stream_lead.py [C|B]"""
import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2509_05464_b200 import _native as N, pipeline as PL, workloads as W
L = N.load()
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C"
w = W.config(cfg); F, A, T, E = w.rf_shape()
rec = PL.Reconstructor(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), keep_lo=2, keep_hi=F, device=dev)
s = torch.cuda.current_stream(dev)
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device=dev)
N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 20260816, s.cuda_stream))
h_rf = torch.empty(w.rf_shape(), dtype=torch.float32, pin_memory=True); h_rf.copy_(d_rf)
h_pd = torch.empty(w.grid.num_points(), dtype=torch.float64, pin_memory=True)
rec.run_resident(d_rf, 3); torch.cuda.synchronize()
K = 5
def timeit(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s); fn(); e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
print(cfg, "resident K=5 ms/step", timeit(lambda: rec.run_resident(d_rf, K)) / K, flush=True)
print("resident K=1 ms", timeit(lambda: rec.run_resident(d_rf, 1)), flush=True)
nz = w.grid.dims[2]
print("das full ms", timeit(lambda: rec.plan.run(d_rf.data_ptr(), 0, nz, rec.x.data_ptr(), rec.work.data_ptr(), None, s.cuda_stream)))
variants = [(1/32, 1/8, 5/16), (1/64, 1/16, 3/16, 1/2), (1/16, 1/4), (1/8, 1/4, 3/8, 1/2, 5/8, 3/4, 7/8)]
for fr in variants:
    if hasattr(rec, "_lead"): del rec._lead
    lead = rec._lead_slabs(fr)
    print(fr, [(kb, ke, hi) for kb, ke, _, hi in lead], flush=True)
    rec.run_pipelined([h_rf], [h_pd]); torch.cuda.synchronize()
    ts = [timeit(lambda: rec.run_pipelined([h_rf] * K, [h_pd] * K)) / K for _ in range(2)]
    t1 = [timeit(lambda: rec.run_pipelined([h_rf], [h_pd])) for _ in range(2)]
    split = timeit(lambda: rec._lead_das(d_rf, rec.x.data_ptr(), s, lead, lambda i, st: None))
    print("  e2e K=5 ms/step", [round(t, 1) for t in ts], "K=1", [round(t, 1) for t in t1], "split DAS (resident)", round(split, 1), flush=True)
