"""Debug harness for the tensor-core Gram: checks the digit planes left in
the work buffer and the Gram against numpy for a small case."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2509_05464_b200 import _native as N  # noqa: E402

F, n = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 64
rng = np.random.default_rng(0)
x = (rng.standard_normal((F, n)) + 1j * rng.standard_normal((F, n))).astype(np.complex64)
ref = x.astype(np.complex128).conj() @ x.astype(np.complex128).T
L = N.load()
dx = torch.from_numpy(np.ascontiguousarray(x).view(np.float32).reshape(F, n, 2)).cuda()
wb = L.fqfg_gram_tc_work_bytes(F)
w = torch.zeros(wb, dtype=torch.uint8, device="cuda")
g = torch.full((F, F, 2), float("nan"), dtype=torch.float64, device="cuda")
N.check(L.fqfg_gram_tc_dev(dx.data_ptr(), F, n, 0, n, g.data_ptr(), w.data_ptr(), 0))
torch.cuda.synchronize()
wh = w.cpu().numpy()
amax = wh[:4 * F].view(np.uint32).view(np.float32)
print("amax", amax[:4], "ref", np.maximum(np.abs(x.real), np.abs(x.imag)).max(1)[:4])
kb = 128 * ((n + 63) // 64)
ao = (4 * F + 255) // 256 * 256
Q = wh[ao:ao + 4 * F * kb].view(np.int8).reshape(4, F, kb).astype(np.float64)
e = np.frexp(amax)[1]
rec = np.zeros((F, kb))
for p in range(4):
    rec += Q[p] * 128.0 ** -(p + 1)
rec *= 2.0 ** e[:, None]
xr = np.zeros((F, kb))
for gi in range((n + 63) // 64):
    cnt = min(64, n - 64 * gi)
    xr[:, 128 * gi:128 * gi + cnt] = x.real[:, 64 * gi:64 * gi + cnt]
    xr[:, 128 * gi + 64:128 * gi + 64 + cnt] = x.imag[:, 64 * gi:64 * gi + cnt]
print("digit reconstruction max rel err", np.abs(rec - xr).max() / np.abs(xr).max())
gg = g.cpu().numpy()
gt = gg[..., 0] + 1j * gg[..., 1]
print("G[0,:4]", gt[0, :4])
print("ref[0,:4]", ref[0, :4])
print("max rel err", np.abs(gt - ref).max() / np.abs(ref).max())
rat = (gt.real / ref.real)
print("ratio re diag", np.diag(rat)[:8])
bad = np.argwhere(~(np.abs(gt - ref) <= 1e-6 * np.abs(ref).max()))
print("bad count", len(bad), "first", bad[:10].tolist(), "rows", sorted(set(bad[:, 0].tolist()))[:20],
      "cols", sorted(set(bad[:, 1].tolist()))[:20])
qb = 4 * F * 128 * ((1 << 21) // 64)
po = ao + (qb + 255) // 256 * 256
mt, nt = (F + 127) // 128, (F + 63) // 64
part = wh[po:po + mt * nt * 128 * 64 * 16].view(np.float64).reshape(mt * nt, 128, 64, 2)
for t in range(mt * nt):
    a, b = divmod(t, nt)
    p = part[t]
    print("tile", t, (a, b), "absmax re", np.abs(p[..., 0]).max(), "nonzero", np.count_nonzero(p[..., 0]))
Fp = (F + 15) // 16 * 16
m0 = 0 if Fp <= 128 else min(128 * 0, Fp - 128)
p = part[1]
print("tile1 row0 cols 0..3 re", p[0, :4, 0], "ref", ref[0, 64:68].real)
for t in range(mt * nt):
    p = part[t]
    badp = np.argwhere(np.abs(p[..., 0]) > 1e5)
    print("tile", t, "garbage entries", len(badp), "rows", sorted(set(badp[:, 0].tolist()))[:12],
          "cols", sorted(set(badp[:, 1].tolist()))[:70])
