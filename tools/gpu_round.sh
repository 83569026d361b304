#!/bin/bash
# One GPU evidence pass: tests, smoke, default bench, ncu launch list + full capture of the TSQR leaf.
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_bench.csv &
CPID=$!
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
kill $CPID
python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tsqr_leaf -c 1 -o gpurun_out/tsqr_leaf_full \
  python tools/run_kernel.py tsqr 2097152 200 1 > gpurun_out/ncu_full.log 2>&1
python tools/run_kernel.py gram 4194304 200 1 > gpurun_out/plain_g.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/gram_full2 \
  python tools/run_kernel.py gram 4194304 200 1 > gpurun_out/ncu_full_g.log 2>&1
python tools/run_kernel.py sketch 1048576 200 1 > gpurun_out/plain_s.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -c 1 -o gpurun_out/skgemm_full \
  python tools/run_kernel.py sketch 1048576 200 1 > gpurun_out/ncu_full_s.log 2>&1
python tools/run_kernel.py tsqr 4194304 25 1 > gpurun_out/plain_n25.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:warp_leaf -c 1 -o gpurun_out/tsqr_warp_leaf_full \
  python tools/run_kernel.py tsqr 4194304 25 1 > gpurun_out/ncu_full_wl.log 2>&1
timeout 900 python bench.py --config C4 --rows 400000000 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C4.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C5.log 2>&1
# summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit)
TSNMF_PROFILE_OUT=gpurun_out/profiles_out python tools/summarize_profiles.py r01 > gpurun_out/summarize.log 2>&1
mkdir -p gpurun_out/reps_keep && mv gpurun_out/tsqr_warp_leaf_full.ncu-rep gpurun_out/reps_keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
echo done
