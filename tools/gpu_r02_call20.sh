#!/bin/bash
mkdir -p gpurun_out/p20
timeout 300 python tools/split_debug2.py > gpurun_out/p20/debug.log 2>&1; echo "rc=$?" >> gpurun_out/p20/debug.log
timeout 600 python tools/split_check.py > gpurun_out/p20/split.log 2>&1; echo "rc=$?" >> gpurun_out/p20/split.log
