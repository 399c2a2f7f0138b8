#!/bin/bash
# Reproduces profiles/r02_k12_chain_probe_nc{4,2}.txt, r02_stepprobe.txt and r02_fpmul_bench.txt (run under gpurun).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k12 tools/k12_chain_probe.cu && /tmp/k12 > gpurun_out/k12.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DK12_NC=2 -o /tmp/k12b tools/k12_chain_probe.cu && /tmp/k12b > gpurun_out/k12_nc2.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_14497_b200/csrc -o /tmp/stepprobe tools/stepprobe.cu && /tmp/stepprobe 2000 > gpurun_out/stepprobe.txt
python tools/fpmul_bench.py > gpurun_out/fpmul.txt
cat gpurun_out/k12.txt gpurun_out/k12_nc2.txt gpurun_out/stepprobe.txt gpurun_out/fpmul.txt
