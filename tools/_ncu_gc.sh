set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_dmma_occ tools/probe_dmma_occ.cu && /tmp/probe_dmma_occ > gpurun_out/probe_dmma_occ.log 2>&1
python tools/run_kernel.py gram 2097152 200 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_cyclic_kernel -c 1 -o gpurun_out/gc12 -f python tools/run_kernel.py gram 2097152 200 1 > gpurun_out/ncu_gc12.log 2>&1
TSNMF_GRAM_CYCLIC=8 ncu --set full --clock-control none --import-source on -k regex:gram_cyclic_kernel -c 1 -o gpurun_out/gc8 -f python tools/run_kernel.py gram 2097152 200 1 > gpurun_out/ncu_gc8.log 2>&1
for r in gc12 gc8; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.summary.txt 2>&1; done
cat gpurun_out/probe_dmma_occ.log gpurun_out/gc12.summary.txt gpurun_out/gc8.summary.txt
