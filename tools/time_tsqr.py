"""Time dv.tsqr with CUDA events (library chosen by TSNMF_LIB_PATH; timing studies only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1402_6964_b200 import device as dv, synthetic
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x = synthetic.generate(synthetic.config("C2", m=m)) if n == 200 else torch.randn(m, n, dtype=torch.float64, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: dv.tsqr(x))
print(f"{os.path.basename(os.environ.get('TSNMF_LIB_PATH', 'default'))}: m={m} n={n} tsqr {ms:.2f} ms {m*n*8/ms/1e6:.1f} GB/s")
