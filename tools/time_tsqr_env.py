"""Time dv.tsqr at the C2 shape (n from argv, default 200; 2^24 rows) under the current environment
(TSNMF_LIB_PATH, TSNMF_SPLIT_CFG, TSNMF_SPLIT_PERM, ...); prints one line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv, synthetic
ns = [int(a) for a in sys.argv[1:]] or [200]
out = []
for n in ns:
    m = 1 << 24
    x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=20))
    xs = x[:50001]
    r = dv.tsqr(xs)[0].cpu().numpy()
    want = np.linalg.qr(xs.cpu().numpy(), mode="r")
    want = want * np.where(np.diagonal(want) < 0, -1.0, 1.0)[:, None]
    err = np.linalg.norm(r - want) / np.linalg.norm(want)
    dv.tsqr(x); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): dv.tsqr(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out.append(f"n={n}: {m * n * 8 / ms / 1e6:.1f} GB/s (R rel {err:.1e})")
    del x; torch.cuda.empty_cache()
tag = " ".join(f"{k[6:]}={v.split('/')[-1]}" for k, v in sorted(os.environ.items()) if k.startswith("TSNMF_"))
print(f"[{tag}] " + "; ".join(out), flush=True)
