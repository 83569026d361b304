#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/split_check.py quick > gpurun_out/c15_split.log 2>&1; echo "rc=$?" >> gpurun_out/c15_split.log
timeout 300 python tools/split_debug2.py > gpurun_out/c15_debug.log 2>&1; echo "rc=$?" >> gpurun_out/c15_debug.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c15_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c15_pytest.log
timeout 600 python tools/fuzz_narrow.py wide > gpurun_out/c15_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/c15_fuzz.log
timeout 300 python tools/trace_split.py 2097152 200 > gpurun_out/c15_trace.log 2>&1
