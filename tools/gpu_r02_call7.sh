#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/split_debug.py > gpurun_out/c7_debug.log 2>&1; echo "rc=$?" >> gpurun_out/c7_debug.log
