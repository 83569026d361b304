#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/split_check.py > gpurun_out/c6_split.log 2>&1; echo "rc=$?" >> gpurun_out/c6_split.log
TSNMF_TSQR_SPLIT=1 timeout 300 python tools/trace_split.py 2097152 200 > gpurun_out/c6_trace.log 2>&1; echo "rc=$?" >> gpurun_out/c6_trace.log
