#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/split_debug2.py > gpurun_out/c10_debug.log 2>&1; echo "rc=$?" >> gpurun_out/c10_debug.log
timeout 600 python tools/split_check.py > gpurun_out/c10_split.log 2>&1; echo "rc=$?" >> gpurun_out/c10_split.log
timeout 900 python -m pytest tests -m gpu -q -x -k "tsqr or factor or stream or parity or tall or combine or column" > gpurun_out/c10_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c10_pytest.log
timeout 600 python tools/fuzz_narrow.py wide > gpurun_out/c10_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/c10_fuzz.log
