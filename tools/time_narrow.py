"""Narrow TSQR leaves (n <= 32): parity vs numpy QR and timing per variant (timing studies only).
Variants are selected by env (read per call): warp-chain leaf (TSNMF_TSQR_WARPLEAF=0) and the
register-block warp leaf with S = 2, 3, 4 rows per lane (TSNMF_WL_S)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1402_6964_b200 import device as dv

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
ns = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [25]
variants = {"chain": {"TSNMF_TSQR_WARPLEAF": "0"}, "wl": {}}


def setenv(kv):
    for k in ("TSNMF_TSQR_WARPLEAF", "TSNMF_WL_S"):
        os.environ.pop(k, None)
    os.environ.update(kv)


def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in ns:
    rng = np.random.default_rng(n)
    xs = rng.uniform(0, 1, (100_003, n)) * np.logspace(0, -2, n)
    want = np.linalg.qr(xs, mode="r")
    want = want * np.where(np.diag(want) < 0, -1.0, 1.0)[:, None]
    xsd = torch.as_tensor(xs, device="cuda")
    x = torch.rand(m, n, dtype=torch.float64, device="cuda")
    for name, kv in variants.items():
        setenv(kv)
        r, l1, sq = dv.tsqr(xsd)
        rel = np.linalg.norm(r.cpu().numpy() - want) / np.linalg.norm(want)
        l1e = np.abs(l1.cpu().numpy() - np.abs(xs).sum(0)).max() / np.abs(xs).sum(0).max()
        ms = t(lambda: dv.tsqr(x))
        plan = dv.tsqr_plan(n, m)
        print(f"n={n} {name}: rel {rel:.2e} l1 {l1e:.1e}  m={m} {ms:.2f} ms {m*n*8/ms/1e6:.1f} GB/s plan {plan}",
              flush=True)
setenv({})
