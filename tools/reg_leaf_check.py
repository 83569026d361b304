"""Register-block TSQR leaf with DMMA trailing updates (tsqr_reg.cu; TSNMF_TSQR_REGLEAF=1): parity vs numpy QR
on ragged / strided shapes for the widths it serves, then timing against the older leaves (=0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv

def ref_r(x):
    r = np.linalg.qr(x, mode="r")
    return r * np.where(np.diagonal(r) < 0, -1.0, 1.0)[:, None]

os.environ["TSNMF_TSQR_REGLEAF"] = "1"
g = np.random.default_rng(0)
worst = 0.0
for n, nt in [(n, nt) for n in list(range(25, 33)) for nt in (8, 10, 12)] + [(n, nt) for n in range(57, 65) for nt in (4, 5, 6)]:
  os.environ["TSNMF_RG_NT"] = str(nt)
  if True:
      for m in [n, n + 1, 100, 257, 4099, 100003, 1 << 20]:
          xh = g.standard_normal((m, n)) * np.logspace(0, -3, n)
          r, l1, sq = dv.tsqr(torch.from_numpy(xh).cuda())
          r = r.cpu().numpy()
          want = ref_r(xh)
          e = np.linalg.norm(r - want) / np.linalg.norm(want)
          el1 = np.abs(l1.cpu().numpy() - np.abs(xh).sum(0)).max() / np.abs(xh).sum(0).max()
          esq = np.abs(sq.cpu().numpy() - (xh * xh).sum(0)).max() / (xh * xh).sum(0).max()
          worst = max(worst, e)
          ok = e < 1e-12 and el1 < 1e-13 and esq < 1e-13 and np.all(np.tril(r, -1) == 0) and np.all(np.diagonal(r) >= 0)
          if not ok:
              print(f"FAIL n={n} m={m} plan={dv.tsqr_plan(n, m)} R rel {e:.2e} l1 {el1:.1e} sq {esq:.1e}", flush=True)
              sys.exit(1)
      xh = g.standard_normal((50000, 80))
      r = dv.tsqr(torch.from_numpy(xh).cuda()[:, 3:3 + n])[0].cpu().numpy()
      e = np.linalg.norm(r - ref_r(xh[:, 3:3 + n])) / np.linalg.norm(ref_r(xh[:, 3:3 + n]))
      assert e < 1e-12, ("strided", n, e)
# nonnegative data with a zero column and a duplicated column (non-unique R: compare R^T R)
xh = g.uniform(0, 1, (30000, 25)); xh[:, 7] = 0.0; xh[:, 9] = xh[:, 3]
r = dv.tsqr(torch.from_numpy(xh).cuda())[0].cpu().numpy()
e = np.linalg.norm(r.T @ r - xh.T @ xh) / np.linalg.norm(xh.T @ xh)
assert e < 1e-12, ("degenerate", e)
print(f"parity ok, worst R rel {worst:.2e}, plan n=25: {dv.tsqr_plan(25, 1 << 24)}", flush=True)
if "quick" in sys.argv:
    sys.exit(0)
for n, m in [(25, 1 << 26), (25, 400_000_000), (32, 1 << 26), (64, 1 << 26), (64, 1 << 28), (57, 1 << 26)]:
    x = torch.rand(m, n, dtype=torch.float64, device="cuda")
    out = []
    for v, nt in [("1", nt) for nt in ((8, 10, 12) if n <= 32 else (4, 5, 6))] + [("0", 0)]:
        os.environ["TSNMF_TSQR_REGLEAF"] = v
        os.environ["TSNMF_RG_NT"] = str(nt)
        dv.tsqr(x); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): dv.tsqr(x)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out.append(f"reg={v} nt={nt}: {m * n * 8 / ms / 1e6:.0f} GB/s")
    print(f"n={n} m={m}: " + "; ".join(out), flush=True)
    del x; torch.cuda.empty_cache()
