#!/bin/bash
# Round-2 evidence pass on one B200 (gpurun): GPU tests, smoke, full-m parity, the bench lines (C2 default,
# C5, one GPU's C4 shard), the reference arm, the split leaf's ncu launch list and --set full summary.
# Outputs under gpurun_out/ev (copy what is judged into profiles/).
set -o pipefail
mkdir -p gpurun_out/ev
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev/smoke.log
timeout 900 python bench.py > gpurun_out/ev/bench_C2.log 2>&1; echo "rc=$?" >> gpurun_out/ev/bench_C2.log
timeout 900 python bench.py --config C5 > gpurun_out/ev/bench_C5.log 2>&1; echo "rc=$?" >> gpurun_out/ev/bench_C5.log
timeout 900 python bench.py --config C4 --rows 400000000 --steps 3 --warmup 3 --no-e2e --k 128 > gpurun_out/ev/bench_C4_shard.log 2>&1; echo "rc=$?" >> gpurun_out/ev/bench_C4_shard.log
timeout 900 python bench.py --impl reference > gpurun_out/ev/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ev/bench_ref.log
[ -n "$PARITY" ] && { timeout 2400 python tests/parity_full.py --configs C2,C3,C5,C4s --out gpurun_out/ev/r02_parity_full.json > gpurun_out/ev/parity.log 2>&1; echo "rc=$?" >> gpurun_out/ev/parity.log; }
python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ev/ncu_launches.log 2>&1
TSNMF_PROFILE_OUT=gpurun_out/ev python tools/summarize_profiles.py r02 > gpurun_out/ev/summ.log 2>&1
echo done
