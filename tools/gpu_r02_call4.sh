#!/bin/bash
mkdir -p gpurun_out
export TSNMF_TSQR_SPLIT=1
python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_leaf -c 1 -o /tmp/split \
  python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c4_ncu.log 2>&1
ncu -i /tmp/split.ncu-rep --page source --csv --print-source sass > gpurun_out/c4_split_sass.csv 2>/dev/null
ncu -i /tmp/split.ncu-rep --page source --csv --print-source cuda > gpurun_out/c4_split_cuda.csv 2>/dev/null
ncu -i /tmp/split.ncu-rep --page raw --csv > gpurun_out/c4_split_raw.csv 2>/dev/null
TSNMF_PROFILE_OUT=gpurun_out python tools/summarize_profiles.py r02 --one /tmp/split.ncu-rep tsqr_split_leaf "split leaf 2^21 x 200" >> gpurun_out/c4_ncu.log 2>&1
gzip -f gpurun_out/c4_split_sass.csv gpurun_out/c4_split_cuda.csv
ls -la gpurun_out
