#!/bin/bash
mkdir -p gpurun_out
echo order1 > gpurun_out/c8_debug.log
TSNMF_SPLIT_ORDER=1 timeout 300 python tools/split_debug2.py >> gpurun_out/c8_debug.log 2>&1
echo miglag1 >> gpurun_out/c8_debug.log
TSNMF_SPLIT_MIGLAG=1 timeout 300 python tools/split_debug2.py >> gpurun_out/c8_debug.log 2>&1
echo both >> gpurun_out/c8_debug.log
TSNMF_SPLIT_MIGLAG=1 TSNMF_SPLIT_ORDER=1 timeout 300 python tools/split_debug2.py >> gpurun_out/c8_debug.log 2>&1
