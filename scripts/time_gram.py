"""Time the Casorati Gram engines at config sizes: FP64 CUDA cores
(fqfg_gram_dev, exact) vs tensor cores (fqfg_gram_tc_dev, int8 digits), on a
synthetic X [F][N] complex64, and their agreement."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05464_b200 import _native as N  # noqa: E402


def main():
    L = N.load()
    cases = [(200, 128 ** 3), (100, 64 ** 3), (400, 256 * 256 * 192)]
    if len(sys.argv) > 1:
        cases = cases[:int(sys.argv[1])]
    for F, n in cases:
        x = torch.randn((F, n, 2), dtype=torch.float32, device="cuda")
        g64 = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
        gtc = torch.empty_like(g64)
        w64 = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
        wtc = torch.empty(L.fqfg_gram_tc_work_bytes(F), dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        res = {}
        for name, fn, g, w in (("fp64", L.fqfg_gram_dev, g64, w64),
                               ("tc", L.fqfg_gram_tc_dev, gtc, wtc)):
            N.check(fn(x.data_ptr(), F, n, 0, n, g.data_ptr(), w.data_ptr(), s))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                N.check(fn(x.data_ptr(), F, n, 0, n, g.data_ptr(), w.data_ptr(), s))
            b.record()
            torch.cuda.synchronize()
            res[name] = a.elapsed_time(b) / 3
        err = ((gtc - g64).abs().max() / g64.abs().max()).item()
        flops = 8.0 * n * F * F
        print(f"F={F} N={n}: fp64 {res['fp64']:.2f} ms, tensor cores {res['tc']:.2f} ms "
              f"({flops / res['tc'] / 1e9:.1f} TF/s useful), max rel diff {err:.2e}", flush=True)
        del x, g64, gtc, w64, wtc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
