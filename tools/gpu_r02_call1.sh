set -o pipefail
mkdir -p gpurun_out
nvidia-smi > gpurun_out/c1_nvsmi.txt 2>&1; nproc >> gpurun_out/c1_nvsmi.txt; free -g >> gpurun_out/c1_nvsmi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/c1_smoke.log
timeout 600 python bench.py > gpurun_out/c1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/c1_bench.log
timeout 2400 python tests/parity_full.py --configs C2,C3,C5,C4s --out gpurun_out/c1_parity_full.json > gpurun_out/c1_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/c1_parity.log
