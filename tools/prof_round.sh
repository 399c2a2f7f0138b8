#!/bin/bash
# Round profiling pass (run under gpurun, 1 GPU): smoke, the default bench line, the ncu launch list of
# the c256 bench, one `ncu --set full` capture each of k_accum and k_tables_coz (c256), the sha of the
# library those captures are of (bench.py reports roofline.traffic only for that build).
CMD="python bench.py --config c256 --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook --no-configs"
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0, '.'); import bench; print(bench.lib_sha16())" > gpurun_out/lib_sha.txt
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
if [ -z "$NO_FULL_BENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
fi
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_accum -s 1 -c 1 -o gpurun_out/prof_accum $CMD > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tables_coz -s 1 -c 1 -o gpurun_out/prof_tables $CMD > gpurun_out/ncu_full_tables.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/smoke.log
