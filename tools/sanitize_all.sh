#!/bin/bash
# compute-sanitizer over tools/sanitize_small.py: memcheck, racecheck, synccheck, initcheck
# (one tool per process); summaries land in gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
# the per-thread Paillier kernels
PCMM_PAILLIER_WARP=0 timeout 900 $CS --tool memcheck python tools/sanitize_small.py paillier > gpurun_out/sanitize_memcheck_paillier_thread.log 2>&1
echo "memcheck(paillier per-thread) rc=$?" >> gpurun_out/sanitize_rc.txt
PCMM_PAILLIER_WARP=0 timeout 900 $CS --tool racecheck python tools/sanitize_small.py paillier > gpurun_out/sanitize_racecheck_paillier_thread.log 2>&1
echo "racecheck(paillier per-thread) rc=$?" >> gpurun_out/sanitize_rc.txt
