"""Phase timing of the TSQR leaf from the trace build (CTA 0, first row block, lane 0 of each warp).
Slots: g_trace[warp][panel*64 + tag] = clock64().  Tags: 1 panel start, 2 panel done, 10+j / 30+j column j
(start / after reduction), 3/4 lookahead start/end, 20..23 GEMM-group stages (last group of the panel)."""
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
buf = np.zeros(8 * 64 * 64, dtype=np.int64)
dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, buf.size)
dv.tsqr(x); torch.cuda.synchronize(); lib.tsnmf_trace_read(buf.ctypes.data, buf.size)
t = buf.reshape(8, 64, 64).astype(np.float64)
P = int((t[0, :, 1] > 0).sum())
print("panels traced:", P, " plan:", dv.tsqr_plan(n, m))
def d(w, p, a, b):
    return t[w, p, b] - t[w, p, a] if t[w, p, a] > 0 and t[w, p, b] > 0 else np.nan
panel = [d(0, p, 1, 2) for p in range(P)]
wait = [t[0, p + 1, 1] - t[0, p, 2] for p in range(P - 1)]
red = np.nanmean([[d(0, p, 10 + j, 30 + j) for j in range(8)] for p in range(P)], axis=0)
upd = np.nanmean([[d(0, p, 30 + j, 10 + j + 1) if j < 7 else d(0, p, 37, 2) for j in range(8)] for p in range(P)], axis=0)
print(f"panel warp: panel {np.nanmean(panel):.0f} clk, wait for ColsReady {np.nanmean(wait):.0f}, first col start {np.nanmean([d(0,p,1,10) for p in range(P)]):.0f}")
print("  per column reduce:", red.astype(int).tolist())
print("  per column update:", upd.astype(int).tolist())
for w in (1, 2, 3, 4, 5, 6, 7):
    la = np.nanmean([d(w, p, 3, 4) for p in range(P)])
    g1 = np.nanmean([d(w, p, 20, 21) for p in range(P)])
    g2 = np.nanmean([d(w, p, 21, 22) for p in range(P)])
    g3 = np.nanmean([d(w, p, 22, 23) for p in range(P)])
    print(f"gemm warp {w}: lookahead {la:.0f}, last group: W {g1:.0f}, T/R {g2:.0f}, B-=VW {g3:.0f}")
lw = 4 if np.nansum(t[4, :, 3]) > 0 else 1
la_start = [t[lw, p, 3] - t[0, p, 2] for p in range(P - 1)]
la_to_panel = [t[0, p + 1, 1] - t[lw, p, 4] for p in range(P - 1)]
print("  per panel: panel done -> lookahead start", [int(v) for v in la_start])
print(f"panel done -> lookahead start {np.nanmean(la_start):.0f}, lookahead end -> next panel start {np.nanmean(la_to_panel):.0f}, panel start -> col0 {np.nanmean([d(0,p,1,10) for p in range(P)]):.0f}, col7 end -> panel done {np.nanmean([d(0,p,37,2) for p in range(P)]):.0f}")
tot = t[0, P - 1, 2] - t[0, 0, 1]
print(f"block span (panel 0 start -> last panel done): {tot:.0f} clk = {tot / P:.0f} per panel")
