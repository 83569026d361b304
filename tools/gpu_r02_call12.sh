#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/split_check.py > gpurun_out/c12_split.log 2>&1; echo "rc=$?" >> gpurun_out/c12_split.log
python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c12_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:split_leaf -c 1 \
  python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/c12_ncu.log 2>&1
