"""Gram with and without the fused column l1 (its cost per width)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1402_6964_b200 import device as dv, synthetic
m = 1 << 23
for n in (200, 64, 25):
    x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=min(20, n)))
    def t(fn, reps=3):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    a = t(lambda: dv.gram(x, stats=True)); b = t(lambda: dv.gram(x, stats=False))
    print(f"n={n}: gram+l1 {m*n*8/a/1e6:.0f} GB/s, gram only {m*n*8/b/1e6:.0f} GB/s")
