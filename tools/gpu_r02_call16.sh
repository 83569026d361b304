#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/split_debug2.py > gpurun_out/c16_debug.log 2>&1; echo "rc=$?" >> gpurun_out/c16_debug.log
timeout 600 python tools/split_check.py > gpurun_out/c16_split.log 2>&1; echo "rc=$?" >> gpurun_out/c16_split.log
timeout 300 python tools/trace_split.py 2097152 200 > gpurun_out/c16_trace.log 2>&1
