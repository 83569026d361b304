#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/split_check.py > gpurun_out/c3_split.log 2>&1; echo "rc=$?" >> gpurun_out/c3_split.log
