"""Shadow-warp timeline from the trace build: per panel, tags 3 (start), 5 (after the block-ready wait),
40+j / 50+j (before / after waiting for reflector j), 4 (done); panel warp tags 10+j (column j start)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["TSNMF_LIB_PATH"] = os.path.join(ROOT, "paper_1402_6964_b200", "libtsnmf_b200_trace.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1402_6964_b200 import _native, device as dv, synthetic
x = synthetic.generate(synthetic.config("C2", m=1 << 20))
lib = _native.load()
lib.tsnmf_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(8 * 64 * 64, dtype=np.int64)
for _ in range(2):
    dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, buf.size)
t = buf.reshape(8, 64, 64).astype(np.float64)
for p in (2, 3, 10):
    base = t[0, p, 1]
    rel = lambda w, tag: (t[w, p, tag] - base) if t[w, p, tag] > 0 else float('nan')
    print(f"panel {p}: panel start 0, col starts", [int(rel(0, 10 + j)) for j in range(8)], "done", int(rel(0, 2)))
    print("   shadow: start", int(rel(4, 3)), "ready", int(rel(4, 5)), "waits", [(int(rel(4, 40 + j)), int(rel(4, 50 + j))) for j in range(8)], "end", int(rel(4, 4)))
