"""Time the GX pieces with CUDA events: full pass, explicit-G GEMM only, G generation only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1402_6964_b200 import device as dv, synthetic
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
k = int(sys.argv[3]) if len(sys.argv) > 3 else 400
x = synthetic.generate(synthetic.config("C2", m=m)) if n == 200 else torch.randn(m, n, dtype=torch.float64, device="cuda")
g = dv.gaussian_rows(0, 0, m, k)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
full = t(lambda: dv.sketch(x, 0, 0, k))
gemm = t(lambda: dv.sketch(x, 0, 0, k, g=g))
gen = t(lambda: dv.gaussian_rows(0, 0, m, k))
fl = 2.0 * k * n * m
print(f"n={n} k={k} full {full:.2f} ms ({m*n*8/full/1e6:.0f} GB/s)  gemm-only {gemm:.2f} ms ({fl/gemm/1e9:.1f} TF/s = {fl/gemm/1e9/37:.2f} of FP64)  gen-only {gen:.2f} ms ({m*k/gen/1e6:.2f} G normals/s)")
