#!/bin/bash
mkdir -p gpurun_out
TSNMF_TSQR_SPLIT=1 timeout 300 python tools/trace_split.py 2097152 200 > gpurun_out/c5_trace.log 2>&1; echo "rc=$?" >> gpurun_out/c5_trace.log
TSNMF_TSQR_SPLIT=0 timeout 300 python tools/trace_tsqr.py 2097152 200 > gpurun_out/c5_trace_old.log 2>&1; echo "rc=$?" >> gpurun_out/c5_trace_old.log
