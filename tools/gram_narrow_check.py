"""Narrow Gram (n <= 64, direct-from-global fragments): parity vs numpy on ragged / strided shapes for every
width, then timing against the staged kernel (TSNMF_GRAM_NARROW=0) and the padded-tile variant (TSNMF_GRAM_TAIL=0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv

g = np.random.default_rng(3)
worst = 0.0
for n in range(1, 65):
    for m in [1, 3, 4, 17, 255, 4099, 100003, 300000]:
        xh = g.standard_normal((m, n)) * np.logspace(0, -2, n)
        G, l1, sq = dv.gram(torch.from_numpy(xh).cuda())
        want = xh.T @ xh
        e = np.linalg.norm(G.cpu().numpy() - want) / np.linalg.norm(want)
        el1 = np.abs(l1.cpu().numpy() - np.abs(xh).sum(0)).max() / np.abs(xh).sum(0).max()
        esq = np.abs(sq.cpu().numpy() - (xh * xh).sum(0)).max() / (xh * xh).sum(0).max()
        worst = max(worst, e, el1, esq)
        assert e < 1e-13 and el1 < 1e-13 and esq < 1e-13, (n, m, e, el1, esq)
        assert np.array_equal(G.cpu().numpy(), G.cpu().numpy().T)
    xh = g.standard_normal((5001, 72))
    xs = torch.from_numpy(xh).cuda()[:, 3:3 + n]
    G = dv.gram(xs)[0].cpu().numpy()
    want = xh[:, 3:3 + n].T @ xh[:, 3:3 + n]
    assert np.linalg.norm(G - want) / np.linalg.norm(want) < 1e-13, ("strided", n)
print(f"parity ok (n = 1..64), worst {worst:.2e}", flush=True)
if "quick" in sys.argv:
    sys.exit(0)

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for n, m in [(64, 1 << 26), (64, 1 << 28), (56, 1 << 26), (48, 1 << 26), (40, 1 << 26), (33, 1 << 26), (32, 1 << 26), (25, 400_000_000)]:
    x = torch.rand(m, n, dtype=torch.float64, device="cuda")
    out = []
    for env in ({}, {"TSNMF_GRAM_TAIL": "0"}, {"TSNMF_GRAM_NARROW": "0"}):
        for k in ("TSNMF_GRAM_TAIL", "TSNMF_GRAM_NARROW"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ms = t(lambda: dv.gram(x))
        out.append(f"{'default' if not env else ','.join(f'{k[11:]}={v}' for k, v in env.items())}: {m * n * 8 / ms / 1e6:.0f} GB/s")
    print(f"n={n} m={m}: " + "; ".join(out), flush=True)
    del x; torch.cuda.empty_cache()
