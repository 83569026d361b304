"""Run one reduction kernel on device-generated C2-like data (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1402_6964_b200 import device as dv, synthetic

op = sys.argv[1] if len(sys.argv) > 1 else "tsqr"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 21
n = int(sys.argv[3]) if len(sys.argv) > 3 else 200
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
spec = synthetic.config("C2", m=m, n=n, r=min(20, n))
x = synthetic.generate(spec)
for _ in range(reps):
    if op == "tsqr":
        dv.tsqr(x)
    elif op == "gram":
        dv.gram(x)
    else:
        dv.sketch(x, 0, 0, 400)
torch.cuda.synchronize()
print("ok", op, m, n)
