"""GX: fused in-CTA generation vs the two-kernel path (TSNMF_SK_FUSED=0) — agreement and timing."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1402_6964_b200 import device as dv
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (m, n, k) in [(1 << 23, 200, 400), (1 << 23, 64, 128), (1 << 23, 25, 128), (100_003, 37, 50)]:
    x = torch.rand(m, n, dtype=torch.float64, device="cuda")
    os.environ["TSNMF_SK_FUSED"] = "0"
    s0 = dv.sketch(x, 12345, 7, k).cpu().numpy(); ms0 = t(lambda: dv.sketch(x, 12345, 7, k))
    os.environ["TSNMF_SK_FUSED"] = "1"
    s1 = dv.sketch(x, 12345, 7, k).cpu().numpy(); ms1 = t(lambda: dv.sketch(x, 12345, 7, k))
    rel = np.linalg.norm(s1 - s0) / np.linalg.norm(s0)
    print(f"m={m} n={n} k={k}: two-kernel {ms0:.2f} ms ({m*n*8/ms0/1e6:.0f} GB/s)  fused {ms1:.2f} ms ({m*n*8/ms1/1e6:.0f} GB/s)  rel {rel:.2e}", flush=True)
