#!/bin/bash
mkdir -p gpurun_out/p19
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/p19/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p19/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p19/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/p19/smoke.log
timeout 2400 python tests/parity_full.py --configs C2,C3,C5,C4s --out gpurun_out/p19/r02_parity_full.json > gpurun_out/p19/parity.log 2>&1; echo "rc=$?" >> gpurun_out/p19/parity.log
