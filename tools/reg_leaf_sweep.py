"""Width sweep n = 25..64: register-block DMMA leaf (TSNMF_TSQR_REGLEAF=1) against the older leaves (=0): parity
vs numpy QR on a ragged shape, then GB/s at 2^25 rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv

g = np.random.default_rng(1)
widths = [int(a) for a in sys.argv[1:]] or list(range(25, 65))
for n in widths:
    xh = g.standard_normal((30011, n)) * np.logspace(0, -3, n)
    want = np.linalg.qr(xh, mode="r"); want *= np.where(np.diagonal(want) < 0, -1.0, 1.0)[:, None]
    m = 1 << 25
    x = torch.rand(m, n, dtype=torch.float64, device="cuda")
    out = []
    for v in ("1", "0"):
        os.environ["TSNMF_TSQR_REGLEAF"] = v
        r = dv.tsqr(torch.from_numpy(xh).cuda())[0].cpu().numpy()
        e = np.linalg.norm(r - want) / np.linalg.norm(want)
        assert e < 1e-12, (n, v, e)
        dv.tsqr(x); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): dv.tsqr(x)
        e1.record(); torch.cuda.synchronize()
        out.append(m * n * 8 / (e0.elapsed_time(e1) / 3) / 1e6)
    print(f"n={n}: reg {out[0]:.0f} GB/s, old {out[1]:.0f} GB/s  ratio {out[0] / out[1]:.2f}", flush=True)
    del x; torch.cuda.empty_cache()
