"""Split-leaf TSQR (256-row blocks, right tiles in L2): parity vs numpy QR and the 128-row leaf, then timing.
python tools/split_check.py [quick]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1402_6964_b200 import device as dv, synthetic

def ref_r(x):
    r = np.linalg.qr(x, mode="r")
    s = np.where(np.diagonal(r) < 0, -1.0, 1.0)
    return r * s[:, None]

def run(x, split):
    os.environ["TSNMF_TSQR_SPLIT"] = "1" if split else "0"
    r, l1, sq = dv.tsqr(x)
    return r.cpu().numpy(), l1.cpu().numpy(), sq.cpu().numpy()

worst = 0.0
g = np.random.default_rng(0)
for n in [105, 112, 127, 150, 199, 200, 208]:
    for m in [n + 1, 257, 1000, 4099, 100003]:
        xh = g.standard_normal((m, n)) * np.logspace(0, -3, n)
        x = torch.from_numpy(xh).cuda()
        r, l1, sq = run(x, True)
        want = ref_r(xh)
        e = np.linalg.norm(r - want) / np.linalg.norm(want)
        el1 = np.abs(l1 - np.abs(xh).sum(0)).max() / np.abs(xh).sum(0).max()
        esq = np.abs(sq - (xh * xh).sum(0)).max() / (xh * xh).sum(0).max()
        worst = max(worst, e)
        print(f"n={n} m={m} plan={dv.tsqr_plan(n, m)} R rel {e:.2e} l1 {el1:.1e} sq {esq:.1e}", flush=True)
        assert e < 1e-12 and el1 < 1e-13 and esq < 1e-13, (n, m)
# strided X (ldx > n) and a non-16-byte-aligned base
xh = g.standard_normal((50000, 210))
x = torch.from_numpy(xh).cuda()[:, 3:203]
r, l1, sq = run(x, True)
e = np.linalg.norm(r - ref_r(xh[:, 3:203])) / np.linalg.norm(ref_r(xh[:, 3:203]))
print("strided", e); assert e < 1e-12
print("worst", worst)
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    sys.exit(0)
for n, m in [(200, 1 << 24), (200, 1 << 26), (128, 1 << 24), (160, 1 << 24), (208, 1 << 24)]:
    spec = synthetic.config("C2", m=m, n=n, r=20)
    x = synthetic.generate(spec)
    for split in (False, True):
        os.environ["TSNMF_TSQR_SPLIT"] = "1" if split else "0"
        dv.tsqr(x); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            dv.tsqr(x)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"n={n} m={m} split={split}: {ms:.2f} ms  {m * n * 8 / ms / 1e6:.1f} GB/s  {2 * n * n * m / ms / 1e9:.2f} TF/s",
              flush=True)
    del x
    torch.cuda.empty_cache()
