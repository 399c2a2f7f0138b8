#!/bin/bash
# ncu --set full capture of one kernel (regex $1) in the c256 bench (run under gpurun)
K=${1:-k_accum}; CFG=${2:-c256}; OUT=${3:-gpurun_out/prof_$K}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$K.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT $CMD > gpurun_out/ncu_$K.log 2>&1
echo "rc=$?"
