#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/trace_split.py 2097152 200 > gpurun_out/c11_trace.log 2>&1
python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c11_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_leaf -c 1 -o /tmp/split \
  python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c11_ncu.log 2>&1
ncu -i /tmp/split.ncu-rep --page source --csv --print-source sass > gpurun_out/c11_split_sass.csv 2>/dev/null
TSNMF_PROFILE_OUT=gpurun_out python tools/summarize_profiles.py r02 --one /tmp/split.ncu-rep tsqr_split_leaf "tsqr_split_leaf_kernel on 2^21 x 200 (tools/run_kernel.py tsqr 2097152 200 1)" >> gpurun_out/c11_ncu.log 2>&1
gzip -f gpurun_out/c11_split_sass.csv
