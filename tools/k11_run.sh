set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k11 tools/k11_imad_probe.cu && /tmp/k11 > gpurun_out/k11.txt 2>&1; cat gpurun_out/k11.txt
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
