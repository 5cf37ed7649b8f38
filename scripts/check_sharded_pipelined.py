"""Functional check of the depth-slab sharded paths (Reconstructor.run_pipelined and run_resident
with a process group: first ensemble streamed in sub-slabs, Gram all-reduce, PD
gather) against the single-GPU step on the same RF.  Several ranks may share one
GPU over gloo (a functional check, not a measurement):
  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/check_sharded_pipelined.py gloo"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_05464_b200 import pipeline as PL, workloads as W  # noqa: E402

backend = sys.argv[1] if len(sys.argv) > 1 else "gloo"
dist.init_process_group(backend)
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0 if backend == "gloo" else rank)
w = W.config("B")
F, A, T, E = w.rf_shape()
rng = np.random.default_rng(3)
rfs = [torch.from_numpy(rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)).pin_memory()
       for _ in range(2)]
rec = PL.Reconstructor(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), keep_lo=2,
                       keep_hi=F, group=dist.group.WORLD)
pds = [torch.zeros(w.grid.num_points(), dtype=torch.float64).pin_memory() for _ in rfs]
rec.run_pipelined(rfs, pds)
torch.cuda.synchronize()
dist.barrier()
# device-resident steps with the cross-ensemble overlap (filter + collectives
# of k on the filter stream during the DAS of k + 1)
d_rf = rfs[1].cuda()
res = rec.run_resident(d_rf, 3)
torch.cuda.synchronize()
res_pd = None if res.pd is None else res.pd.cpu().numpy()
dist.barrier()
if rank == 0:
    one = PL.Reconstructor(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), keep_lo=2,
                           keep_hi=F)
    for k, h in enumerate(rfs):
        want = one.step(h.cuda()).pd.cpu().numpy()
        got = pds[k].numpy()
        rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        print(f"ensemble {k}: world {world}, lead sub-slabs {len(rec._lead)}, PD rel-L2 vs one GPU "
              f"{rel:.2e}", flush=True)
        assert rel < 1e-9, rel
        if k == 1:
            rel = float(np.linalg.norm(res_pd - want) / np.linalg.norm(want))
            print(f"run_resident x3: PD rel-L2 vs one GPU {rel:.2e}", flush=True)
            assert rel < 1e-9, rel
    print("sharded run_pipelined / run_resident OK")
dist.destroy_process_group()
