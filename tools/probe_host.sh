#!/bin/bash
# Host + GPU facts for the design notes (cores, RAM, clocks, DGEMM, pinned H2D).
set -x
nproc; lscpu | head -20; free -g; nvidia-smi; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"
./tools/probe_fp64
python - << 'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): c = a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("cuBLAS DGEMM 8192^3: %.2f TFLOP/s" % (2 * 8192**3 / ms / 1e9))
h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory(); d = torch.empty(1 << 30, dtype=torch.uint8, device='cuda')
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); e0.record()
for _ in range(5): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("pinned H2D 1 GiB: %.1f GB/s" % (5 * (1 << 30) / e0.elapsed_time(e1) / 1e6))
t = time.time(); big = torch.empty(32 << 30, dtype=torch.uint8).pin_memory(); print("pin 32 GiB took %.1f s" % (time.time() - t))
PY
