#!/bin/bash
# round 2, call 2: tests (incl. the reference-backend tests), full-m parity, bench (+ reference arm),
# n=64 leaf ncu capture, then compute-sanitizer racecheck on the leaves / Gram / sketch.
set -o pipefail
mkdir -p gpurun_out/p
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_pytest_gpu.log
timeout 2400 python tests/parity_full.py --configs C2,C3,C5,C4s --out gpurun_out/c2_parity_full.json > gpurun_out/c2_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/c2_parity.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv -lms 1000 > gpurun_out/c2_clocks.csv &
CP=$!
timeout 900 python bench.py > gpurun_out/c2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/c2_bench.log
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/c2_bench_C5.log 2>&1; echo "rc=$?" >> gpurun_out/c2_bench_C5.log
kill $CP
timeout 900 python bench.py --impl reference > gpurun_out/c2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/c2_bench_ref.log
# n = 64 leaf (C5 width): full capture -> summary (the .ncu-rep stays on the box)
python tools/run_kernel.py tsqr 2097152 64 1 > gpurun_out/c2_plain64.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsqr_leaf -c 1 -o /tmp/leaf64 \
  python tools/run_kernel.py tsqr 2097152 64 1 > gpurun_out/c2_ncu64.log 2>&1 && \
  TSNMF_PROFILE_OUT=gpurun_out/p python tools/summarize_profiles.py r02 --one /tmp/leaf64.ncu-rep tsqr_leaf_n64 \
  "tsqr_leaf_kernel (three 4-warp CTAs / SM) on 2^21 x 64 (C5 width; tools/run_kernel.py tsqr 2097152 64 1)" >> gpurun_out/c2_ncu64.log 2>&1
# racecheck (one tool this call); small sizes
for a in "tsqr 65536 200" "tsqr 65536 64" "tsqr 262144 25" "gram 65536 200" "gram 65536 25" "sketch 65536 200"; do
  set -- $a
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/run_kernel.py $1 $2 $3 1 \
    > gpurun_out/p/r02_racecheck_$1_n$3.log 2>&1; echo "rc=$?" >> gpurun_out/p/r02_racecheck_$1_n$3.log
done
echo done
