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
# --set full captures of the kernels new in round 2 (each after its plain run exited 0); summaries only travel back
cap() {  # cap NAME KERNEL_REGEX DESC -- run_kernel args
  local name=$1 rx=$2 desc=$3; shift 3
  python tools/run_kernel.py "$@" > gpurun_out/ev/plain_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 -o gpurun_out/ev/$name -f \
    python tools/run_kernel.py "$@" > gpurun_out/ev/ncu_$name.log 2>&1 && \
  TSNMF_PROFILE_OUT=gpurun_out/ev python tools/summarize_profiles.py r02 --one gpurun_out/ev/$name.ncu-rep $name "$desc" \
    > gpurun_out/ev/summ_$name.log 2>&1
  rm -f gpurun_out/ev/$name.ncu-rep
}
cap tsqr_split_leaf tsqr_split_leaf "tsqr_split_leaf_kernel on 2^21 x 200 (tools/run_kernel.py tsqr 2097152 200 1)" tsqr 2097152 200 1
cap gram_cyclic gram_cyclic "gram_cyclic_kernel<8,3> on 2^22 x 200 (C2 width; tools/run_kernel.py gram 4194304 200 1)" gram 4194304 200 1
cap gram_narrow_n25 gram_narrow "gram_narrow_kernel<3,1> on 2^24 x 25 (C4 width; tools/run_kernel.py gram 16777216 25 1)" gram 16777216 25 1
cap gram_narrow_n64 gram_narrow "gram_narrow_kernel<8,0> on 2^22 x 64 (C5 width; tools/run_kernel.py gram 4194304 64 1)" gram 4194304 64 1
cap tsqr_reg_leaf_n64 tsqr_reg_leaf "tsqr_reg_leaf_kernel<8,6> on 2^21 x 64 (C5 width; tools/run_kernel.py tsqr 2097152 64 1)" tsqr 2097152 64 1
cap tsqr_warp_leaf tsqr_warp_leaf "tsqr_warp_leaf_kernel<25,3> on 2^22 x 25 (C4 width; tools/run_kernel.py tsqr 4194304 25 1)" tsqr 4194304 25 1
cap sketch_gemm sketch_gemm "sketch_gemm_kernel (fused generation) on 2^20 x 200, k = 400 (tools/run_kernel.py sketch 1048576 200 1)" sketch 1048576 200 1
echo done
