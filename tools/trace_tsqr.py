"""Phase timing of the TSQR leaf (CTA 0) with the instrumented library (make -C csrc trace)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["TSNMF_LIB_PATH"] = os.path.join(ROOT, "paper_1402_6964_b200", "libtsnmf_b200_trace.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1402_6964_b200 import _native, device as dv, synthetic
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=min(20, n)))
lib = _native.load()
lib.tsnmf_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(1 << 16, dtype=np.int64)
dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, 1 << 16)
dv.tsqr(x); torch.cuda.synchronize()
k = lib.tsnmf_trace_read(buf.ctypes.data, 1 << 16)
ev = buf[:k].reshape(-1, 2)
panel, gemm, load, blocks = [], [], [], 0
for i in range(len(ev) - 1):
    tag, t = ev[i]; nt = ev[i + 1][1]
    if tag == 0: load.append(nt - t); blocks += 1
    elif tag == 1: panel.append(nt - t)
    elif tag == 2: gemm.append(nt - t)
print(f"blocks {blocks}  panels {len(panel)}")
print(f"per panel: panel-warp phase {np.mean(panel):.0f} clk (median {np.median(panel):.0f}), gemm phase {np.mean(gemm):.0f} clk")
print(f"per block: load+stats {np.mean(load):.0f}, total {(ev[-1][1]-ev[0][1])/max(blocks,1):.0f} clk")
g = np.array(gemm[:25]); print("gemm by panel (first block):", g.astype(int).tolist())
p = np.array(panel[:25]); print("panel by panel (first block):", p.astype(int).tolist())
