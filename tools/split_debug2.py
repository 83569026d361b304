import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1402_6964_b200 import device as dv
g = np.random.default_rng(0)
def ref_r(x):
    r = np.linalg.qr(x, mode="r"); return r * np.where(np.diagonal(r) < 0, -1.0, 1.0)[:, None]
for n, m in [(200, 256), (200, 200), (200, 255), (200, 300), (105, 256), (105, 512), (105, 106), (105, 250),
             (200, 100003), (200, 1 << 20), (160, 1 << 20)]:
    xh = g.standard_normal((m, n)); x = torch.from_numpy(xh).cuda()
    r = dv.tsqr(x)[0].cpu().numpy(); want = ref_r(xh)
    same = all(np.array_equal(r, dv.tsqr(x)[0].cpu().numpy()) for _ in range(3))
    e = np.linalg.norm(r - want) / np.linalg.norm(want)
    print(f"{os.environ.get('TSNMF_LIB_PATH','main')[-12:]} n={n} m={m} plan={dv.tsqr_plan(n, m)} err {e:.2e} deterministic {same}", flush=True)
