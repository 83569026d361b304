"""Ingest path timing: file -> ChunkReader(device) -> stream_pass, against the raw
sequential read of the same file and the device finiteness scan alone.  argv: rows n path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1402_6964_b200 as tb
from paper_1402_6964_b200 import device as dv, synthetic
from paper_1402_6964_b200.matio import HEADER_BYTES, _HDR

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
path = sys.argv[3] if len(sys.argv) > 3 else "/tmp/tsnmf_ingest.bin"
x = synthetic.generate(synthetic.config("C2", m=m, n=n, r=min(20, n)))
with open(path, "wb") as f:  # reference binary layout, written in slabs
    f.write(_HDR.pack(b"TS", 1, m, n))
    for o in range(0, m, 1 << 20):
        f.write(x[o:o + (1 << 20)].cpu().numpy().astype("<f8").tobytes())
gb = m * n * 8 / 1e9
torch.cuda.synchronize()
t0 = time.perf_counter()
with open(path, "rb") as f:
    buf = bytearray(1 << 28)
    while f.readinto(buf):
        pass
t_read = time.perf_counter() - t0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dv.first_nonfinite(x); e0.record(); dv.first_nonfinite(x); e1.record(); torch.cuda.synchronize()
t_scan = e0.elapsed_time(e1) / 1e3
torch.cuda.synchronize(); t0 = time.perf_counter()
rd = tb.ChunkReader(path, device="cuda")
t_init = time.perf_counter() - t0
for ch in rd:
    pass
torch.cuda.synchronize(); t_rd = time.perf_counter() - t0
print(f"reader alone: {gb / t_rd:6.2f} GB/s ({t_rd:.2f} s incl. {t_init:.2f} s setup)", flush=True)
from paper_1402_6964_b200 import gds
cases = [("device", dict(device="cuda")), ("host chunks", dict())]
if gds.available():
    cases.insert(1, ("device, cuFile", dict(device="cuda", gds=True)))
for label, kw in cases:
    if kw.get("gds"):
        tb.stream_pass(tb.ChunkReader(path, **kw))  # first use opens the cuFile driver (not timed)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = tb.stream_pass(tb.ChunkReader(path, **kw))
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"{label:14s}: {gb / t:6.2f} GB/s ({t:.2f} s, rows {res.rows}, chunks {res.chunks})", flush=True)
print(f"raw sequential read {gb / t_read:.2f} GB/s; device finiteness scan {gb / t_scan:.0f} GB/s "
      f"({m} x {n}, {gb:.1f} GB)")
os.remove(path)
