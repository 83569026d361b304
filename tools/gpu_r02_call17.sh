#!/bin/bash
# evidence for the split leaf: bench C2 (+ launch list under ncu) and one --set full capture
mkdir -p gpurun_out/p17
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv -lms 1000 > gpurun_out/p17/clocks.csv &
CP=$!
timeout 900 python bench.py > gpurun_out/p17/bench_C2.log 2>&1; echo "rc=$?" >> gpurun_out/p17/bench_C2.log
kill $CP
python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/p17/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/p17/ncu_launches.log 2>&1
python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/p17/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_leaf -c 1 -o /tmp/split \
  python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/p17/ncu_full.log 2>&1
TSNMF_PROFILE_OUT=gpurun_out/p17 python tools/summarize_profiles.py r02 --one /tmp/split.ncu-rep tsqr_split_leaf "tsqr_split_leaf_kernel on 2^21 x 200 (tools/run_kernel.py tsqr 2097152 200 1)" >> gpurun_out/p17/ncu_full.log 2>&1
TSNMF_PROFILE_OUT=gpurun_out/p17 python tools/summarize_profiles.py r02 > gpurun_out/p17/summ.log 2>&1
