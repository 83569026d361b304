"""Cyclic register Gram (n = 193..200): parity vs numpy on ragged / strided shapes, then C2-shape timing against
the staged kernel (TSNMF_GRAM_CYCLIC=0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv, synthetic

g = np.random.default_rng(5)
worst = 0.0
for variant in ("12", "8"):
  os.environ["TSNMF_GRAM_CYCLIC"] = variant
  for n in range(193, 201):
      for m in [1, 5, 255, 4099, 100003]:
          xh = g.standard_normal((m, n)) * np.logspace(0, -2, n)
          G, l1, sq = dv.gram(torch.from_numpy(xh).cuda())
          want = xh.T @ xh
          e = np.linalg.norm(G.cpu().numpy() - want) / np.linalg.norm(want)
          emax = np.abs(G.cpu().numpy() - want).max() / np.abs(want).max()
          el1 = np.abs(l1.cpu().numpy() - np.abs(xh).sum(0)).max() / np.abs(xh).sum(0).max()
          esq = np.abs(sq.cpu().numpy() - (xh * xh).sum(0)).max() / (xh * xh).sum(0).max()
          worst = max(worst, e, el1, esq)
          assert e < 1e-13 and emax < 1e-13 and el1 < 1e-13 and esq < 1e-13, (n, m, e, emax, el1, esq)
          assert np.array_equal(G.cpu().numpy(), G.cpu().numpy().T)
      xh = g.standard_normal((5001, 210))
      xs = torch.from_numpy(xh).cuda()[:, 3:3 + n]
      G = dv.gram(xs)[0].cpu().numpy()
      want = xh[:, 3:3 + n].T @ xh[:, 3:3 + n]
      assert np.linalg.norm(G - want) / np.linalg.norm(want) < 1e-13, ("strided", n)
print(f"parity ok (n = 193..200), worst {worst:.2e}", flush=True)
if "quick" in sys.argv:
    sys.exit(0)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for n, m in [(200, 1 << 24), (200, 1 << 26), (193, 1 << 24)]:
    x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=20))
    out = []
    for env in ({"TSNMF_GRAM_CYCLIC": "12"}, {"TSNMF_GRAM_CYCLIC": "8"}, {"TSNMF_GRAM_CYCLIC": "0"}):
        os.environ.pop("TSNMF_GRAM_CYCLIC", None)
        os.environ.update(env)
        ms = t(lambda: dv.gram(x))
        out.append(f"{env['TSNMF_GRAM_CYCLIC']}: {m * n * 8 / ms / 1e6:.0f} GB/s = {m * n * (n + 1) / ms / 1e9:.1f} TF/s")
    print(f"n={n} m={m}: " + "; ".join(out), flush=True)
    del x; torch.cuda.empty_cache()
