#!/bin/bash
# Round profiling pass (run under gpurun, 1 GPU): smoke, plain bench, launch list,
# one `ncu --set full` capture each of k_accum, k_tables_fast and k_affine on the c256 bench.
CMD="python bench.py --config c256 --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook"
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_accum -s 1 -c 1 -o gpurun_out/prof_accum $CMD > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tables_fast -s 1 -c 1 -o gpurun_out/prof_tables $CMD > gpurun_out/ncu_full_tables.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_affine -s 1 -c 1 -o gpurun_out/prof_affine $CMD > gpurun_out/ncu_full_affine.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/smoke.log
