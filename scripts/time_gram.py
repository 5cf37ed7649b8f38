"""Time the Casorati Gram (fqfg_gram_dev) for each FP64 tile size (FQFG_GRAM_TB)
the FP64 tensor-core (DMMA) engine and the tcgen05 3xTF32 engine on X [F][N] (config C: F = 200, N = 128^3);
prints ms and the max deviation from the 64-tile result.  Not a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_05464_b200 import _native as N  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 200
NV = int(sys.argv[2]) if len(sys.argv) > 2 else 128 ** 3
L = N.load()
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randn((F, NV, 2), device="cuda", generator=g) * torch.logspace(
    0, -3, NV, device="cuda")[None, :, None]
gram = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
work = torch.empty(256 * F * F * 16, dtype=torch.uint8, device="cuda")
ref = None
for tb in sys.argv[3:] or ["64", "48", "40", "32", "tc"]:
    os.environ.pop("FQFG_GRAM", None)
    if tb in ("tc", "dmma"):
        os.environ["FQFG_GRAM"] = tb
    else:
        os.environ["FQFG_GRAM_TB"] = tb
    run = lambda: N.check(L.fqfg_gram_dev(x.data_ptr(), F, NV, 0, NV, gram.data_ptr(),  # noqa
                                          work.data_ptr(), None))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    if ref is None:
        ref = gram.clone()
    d = float((gram - ref).abs().max() / ref.abs().max())
    useful = F * (F + 1) / 2 * NV * 8
    print(f"F={F} N={NV} tile={tb}: {ms:.2f} ms  {useful / ms / 1e9:.1f} useful TF/s  "
          f"maxdev {d:.1e}", flush=True)
