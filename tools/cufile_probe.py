"""Step-by-step probe of the cuFile binding (gds.py) on this box: driver open, handle registration, reads from
the main thread and from a worker thread, small and large, aligned and unaligned offsets."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(45, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
from paper_1402_6964_b200 import gds

def log(*a):
    print(*a, flush=True)

path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/cufile_probe.bin"
nbytes = int(sys.argv[2]) if len(sys.argv) > 2 else 64 << 20
data = np.random.default_rng(0).integers(0, 255, nbytes + 16, dtype=np.uint8)
data.tofile(path)
log("file written", nbytes + 16)
torch.cuda.init(); torch.zeros(1, device="cuda")
log("available", gds.available())
t0 = time.perf_counter(); fh = gds.FileHandle(path); log("handle registered, O_DIRECT =", fh.direct, f"{time.perf_counter() - t0:.3f}s")
buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for off, size in ((0, 4096), (16, 4096), (16, 1 << 20), (16, nbytes)):
    t0 = time.perf_counter(); got = fh.read_into(buf.data_ptr(), size, off); dt = time.perf_counter() - t0
    ok = bool((buf[:size].cpu().numpy() == data[off:off + size]).all())
    log(f"main thread: offset {off} size {size}: got {got} in {dt:.3f}s ({size / dt / 1e9:.2f} GB/s) correct={ok}")
with ThreadPoolExecutor(max_workers=1) as pool:
    ev = torch.cuda.Event(); ev.record()
    def work():
        ev.synchronize()
        with torch.cuda.device(0):
            return fh.read_into(buf.data_ptr(), nbytes, 16)
    t0 = time.perf_counter(); got = pool.submit(work).result(); dt = time.perf_counter() - t0
    log(f"worker thread: got {got} in {dt:.3f}s ({nbytes / dt / 1e9:.2f} GB/s) correct={bool((buf.cpu().numpy() == data[16:16 + nbytes]).all())}")
fh.close()
os.remove(path)
log("done")
