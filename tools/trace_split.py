"""Per-panel clock64 timeline of the split TSQR leaf (CTA 0, second 256-row block) from the trace build
(make -C paper_1402_6964_b200/csrc trace).  python tools/trace_split.py [m] [n]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["TSNMF_LIB_PATH"] = os.path.join(ROOT, "paper_1402_6964_b200", "libtsnmf_b200_trace.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1402_6964_b200 import _native, device as dv, synthetic
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=min(20, n)))
lib = _native.load()
lib.tsnmf_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(8 * 64 * 64, dtype=np.int64)
dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, buf.size)
dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, buf.size)
t = buf.reshape(8, 64, 64)
t0 = t[0, 0, 41]
npan = (n + 7) // 8
print("panel | P:start panel_done look_done | H:got_panel look_done | GEMM warps (6=got panel, 7=smem done, 8=global done)")
prev = None
for p in range(npan):
    P = [t[0, p, k] - t0 if t[0, p, k] else -1 for k in (41, 42, 45)]
    H = [t[4, p, k] - t0 if t[4, p, k] else -1 for k in (43, 44)]
    G = []
    for w in (1, 2, 3, 5, 6, 7):
        G.append(tuple(int(t[w, p, k] - t0) if t[w, p, k] else -1 for k in (46, 47, 48)))
    gend = max(max(g) for g in G)
    dur = P[0] - prev if prev is not None else 0
    prev = P[0]
    print(f"{p:3d} | {P} (panel {P[1]-P[0]}, look {P[2]-P[1]}) | {H} | gemm end {gend}  step {dur}")
    print("      ", G)
