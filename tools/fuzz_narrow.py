"""Randomised parity sweep of the TSQR leaves against numpy QR: ragged m, strided X; argv[1] = "wide" for
n = 33..256 (panel leaf) instead of n = 1..32 (warp leaf)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1402_6964_b200 import device as dv
rng = np.random.default_rng(2026)
worst = 0.0
wide = len(sys.argv) > 1 and sys.argv[1] == "wide"
cases = 60 if wide else 300
for it in range(cases):
    n = int(rng.integers(33, 257)) if wide else int(rng.integers(1, 33))
    m = int(rng.choice([n, n + 1, 33, 95, 96, 97, 127, 128, 129, 1000, 4097, int(rng.integers(n, 300_000))]))
    ld = n + int(rng.choice([0, 0, 0, 1, 3]))
    full = rng.standard_normal((m, ld)) * rng.choice([1e-3, 1.0, 1e3])
    x = np.ascontiguousarray(full[:, :n])
    xd = torch.as_tensor(full, device="cuda")[:, :n]
    r, l1, sq = dv.tsqr(xd)
    r = r.cpu().numpy()
    if m >= n:
        want = np.linalg.qr(x, mode="r"); want = want * np.where(np.diag(want) < 0, -1.0, 1.0)[:, None]
        err = np.linalg.norm(r - want) / max(np.linalg.norm(want), 1e-300)
    else:
        err = np.linalg.norm(r.T @ r - x.T @ x) / max(np.linalg.norm(x.T @ x), 1e-300)
    e1 = np.abs(l1.cpu().numpy() - np.abs(x).sum(0)).max() / max(np.abs(x).sum(0).max(), 1e-300)  # stats too
    worst = max(worst, err)
    if err > 1e-10 or e1 > 1e-12 or not np.isfinite(err):
        print("FAIL", it, n, m, ld, err, e1); sys.exit(1)
print(f"ok {cases} cases ({'wide' if wide else 'narrow'}), worst R rel", worst)
