"""Time the DAS kernel for several kernel shapes (J, VPW, NW) on a workload.
Prints DAS ms/step (CUDA events around the kernel), never a bench number."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_05464_b200 import _native as N, pipeline as PL, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "B"
# each shape: version:J:VPW:NW[:EB[:MODE[:NS[:PAIRY[:PW[:HINT_NS[:PF]]]]]]]
shapes = [tuple(int(x) for x in s.split(":")) for s in sys.argv[2:]] or [(2, 7, 8, 8, 4)]
w = W.config(cfg)
F, A, T, E = w.rf_shape()
d_rf = torch.empty(w.rf_shape(), dtype=torch.float32, device="cuda")
L = N.load()
N.check(L.fqfg_synth_rf_dev(d_rf.data_ptr(), d_rf.numel(), 1, 0))
pairs = PL.active_pairs_per_plane(w.grid, w.elements, 1.5).sum() * A * F
ref = None
for shp in shapes:
    ver, J, VPW, NW = shp[:4]
    EB = shp[4] if len(shp) > 4 else 4
    MODE = shp[5] if len(shp) > 5 else 0
    NS = shp[6] if len(shp) > 6 else 2
    PY = shp[7] if len(shp) > 7 else 0
    PW = shp[8] if len(shp) > 8 else 4
    HINT = shp[9] if len(shp) > 9 else 0
    PF = shp[10] if len(shp) > 10 else 0
    os.environ["FQFG_DAS_PF"] = str(PF)
    os.environ.update(FQFG_DAS_PAIRY=str(PY), FQFG_DAS_PW=str(PW), FQFG_DAS_HINT=str(HINT),
                      FQFG_DAS_KERNEL=str(ver), FQFG_DAS_J=str(J), FQFG_DAS_VPW=str(VPW),
                      FQFG_DAS_NW=str(NW), FQFG_DAS_EB=str(EB), FQFG_DAS_MODE=str(MODE),
                      FQFG_DAS_NS=str(NS))
    plan = PL.DasPlan(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf())
    x = torch.empty((F, w.grid.num_points(), 2), dtype=torch.float32, device="cuda")
    work = torch.empty(plan.work_bytes, dtype=torch.uint8, device="cuda")
    plan.run(d_rf.data_ptr(), 0, w.grid.dims[2], x.data_ptr(), work.data_ptr())
    L.fqfg_das_plan_set_timing(plan.handle, 1)
    for _ in range(3):
        plan.run(d_rf.data_ptr(), 0, w.grid.dims[2], x.data_ptr(), work.data_ptr())
    dm, da = C.c_double(), C.c_double()
    N.check(L.fqfg_das_last_timing(plan.handle, dm, da))
    torch.cuda.synchronize()
    if ref is None:
        ref = x.clone()
    err = float((x - ref).abs().max() / ref.abs().max())
    das = da.value / 3
    print(f"{cfg} v{ver}m{MODE}s{NS}y{PY}p{PW}h{HINT}pf{PF} J={J} VPW={VPW} NW={NW} EB={EB} tile={plan.tile} "
          f"passes={plan.n_passes} das {das:.2f} ms demod {dm.value / 3:.2f} ms  "
          f"{pairs / das / 1e9:.3f} T active samples/s  gather-equiv "
          f"{16 * pairs / das / 1e6:.0f} GB/s  maxdiff {err:.1e}", flush=True)
    del plan
