"""Time the filter stages (Gram, eig, projection+PD) on a synthetic ensemble."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2509_05464_b200 import _native as N  # noqa: E402

L = N.load()
for F, nvox in [(100, 64**3), (200, 128**3)]:
    x = torch.randn((F, nvox, 2), device="cuda", dtype=torch.float32)
    g = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
    w = torch.empty(F, dtype=torch.float64, device="cuda")
    v = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
    pd = torch.empty(nvox, dtype=torch.float64, device="cuda")
    work = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    def t(fn, n=3):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    os.environ["FQFG_GRAM"] = "tc"
    ttc = t(lambda: N.check(L.fqfg_gram_dev(x.data_ptr(), F, nvox, 0, nvox, g.data_ptr(), work.data_ptr(), s)))
    gtc = g.clone()
    os.environ["FQFG_GRAM"] = "fp64"
    tg = t(lambda: N.check(L.fqfg_gram_dev(x.data_ptr(), F, nvox, 0, nvox, g.data_ptr(), work.data_ptr(), s)))
    rel = float((gtc - g).abs().max() / g.abs().max())
    print(f"F={F} N={nvox}: gram tcgen05 {ttc:.2f} ms (max rel diff vs FP64 {rel:.1e})")
    g0 = g.clone()
    def eig():
        g.copy_(g0)
        N.check(L.fqfg_eig_dev(g.data_ptr(), F, w.data_ptr(), v.data_ptr(), s))
    te = t(eig)
    tp = t(lambda: N.check(L.fqfg_project_pd_dev(x.data_ptr(), F, nvox, 0, nvox, v.data_ptr(), 2, F, None, pd.data_ptr(), s)))
    tp2 = t(lambda: N.check(L.fqfg_project_pd_dev(x.data_ptr(), F, nvox, 0, nvox, v.data_ptr(), 5, F // 2, None, pd.data_ptr(), s)))
    print(f"F={F} N={nvox}: gram {tg:.2f} ms  eig {te:.2f} ms  project(rank1) {tp:.2f} ms  project(full) {tp2:.2f} ms")
