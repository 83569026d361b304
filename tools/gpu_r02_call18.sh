#!/bin/bash
mkdir -p gpurun_out/p18
timeout 600 python -m pytest tests/test_gpu_reduced.py -q -x > gpurun_out/p18/pytest_reduced.log 2>&1; echo "rc=$?" >> gpurun_out/p18/pytest_reduced.log
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/p18/bench_C5.log 2>&1; echo "rc=$?" >> gpurun_out/p18/bench_C5.log
timeout 900 python bench.py --config C4 --rows 400000000 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p18/bench_C4.log 2>&1; echo "rc=$?" >> gpurun_out/p18/bench_C4.log
