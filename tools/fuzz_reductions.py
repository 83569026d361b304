"""Randomised parity sweep of the Gram and GX kernels (ragged m, strided X, random widths, k, row offsets,
seeds) against numpy with the device generator's own G (and the fused vs two-kernel GX paths)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv

rng = np.random.default_rng(77)
worst_g = worst_s = 0.0
for it in range(80):
    n = int(rng.choice([int(rng.integers(1, 40)), int(rng.integers(40, 260)), int(rng.integers(260, 513))]))
    m = int(rng.choice([1, 7, 33, 100, 1000, 40_000, int(rng.integers(1, 200_000))]))
    ld = n + int(rng.choice([0, 0, 1, 5]))
    full = rng.standard_normal((m, ld))
    x = np.ascontiguousarray(full[:, :n])
    xd = torch.as_tensor(full, device="cuda")[:, :n]
    g, l1, sq = dv.gram(xd)
    want = x.T @ x
    eg = np.linalg.norm(g.cpu().numpy() - want) / max(np.linalg.norm(want), 1e-300)
    el = np.abs(l1.cpu().numpy() - np.abs(x).sum(0)).max() / max(np.abs(x).sum(0).max(), 1e-300)
    worst_g = max(worst_g, eg)
    if eg > 1e-12 or el > 1e-12:
        print("GRAM FAIL", it, m, n, ld, eg, el); sys.exit(1)
    if n <= 256 and m <= 50_000:
        k = int(rng.integers(1, 160)); off = int(rng.integers(0, 1 << 40)); seed = int(rng.integers(0, 1 << 32))
        gm = dv.gaussian_rows(seed, off, m, k).cpu().numpy()
        sw = gm.T @ x
        for fused in ("1", "0"):
            os.environ["TSNMF_SK_FUSED"] = fused
            s = dv.sketch(xd, off, seed, k).cpu().numpy()
            es = np.linalg.norm(s - sw) / max(np.linalg.norm(sw), 1e-300)
            worst_s = max(worst_s, es)
            if es > 1e-12:
                print("SKETCH FAIL", it, m, n, ld, k, off, seed, fused, es); sys.exit(1)
        os.environ.pop("TSNMF_SK_FUSED")
print(f"ok 80 cases: worst Gram rel {worst_g:.2e}, worst sketch rel {worst_s:.2e}")
