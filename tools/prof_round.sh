#!/bin/bash
# Profiling pass (run under gpurun): plain bench, launch list, one full capture of k_accum.
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook"
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_accum -s 1 -c 1 -o gpurun_out/prof_accum $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/smoke.log
