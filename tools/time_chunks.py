"""stream_pass over many device RowChunks vs one resident chunk (per-chunk overhead of the host engine)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_6964_b200 as tb
from paper_1402_6964_b200 import synthetic
m = 1 << 23
x = synthetic.generate(synthetic.config("C2", m=m))
for rows in (m, 1 << 20, 1 << 16, 8192):
    chunks = [tb.RowChunk(o, x[o:o + rows]) for o in range(0, m, rows)]
    tb.stream_pass(chunks[:2]); torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tb.stream_pass(chunks)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"chunk rows {rows:8d} ({len(chunks):5d} chunks): {dt*1e3:8.1f} ms  {m*200*8/dt/1e9:6.1f} GB/s  depth {res.tree_depth}")
