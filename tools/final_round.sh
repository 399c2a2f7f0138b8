#!/bin/bash
# Round-end measurement pass (run under gpurun): profile round (smoke, full bench line, ncu launch
# list, ncu --set full captures), the t = 4, 8 rows of the (n, t) grid, the ML ncu capture of k_tables_coz.
bash tools/prof_round.sh > gpurun_out/prof_round.log 2>&1
python tools/grid.py 4,8,12,16 64,256,512 > gpurun_out/grid_t48.md 2> gpurun_out/grid_t48.err
python tools/vector_grid.py > gpurun_out/vector_grid.md 2> gpurun_out/vector_grid.err
CMDML="python bench.py --config ml --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook --no-configs"
ncu --set full --clock-control none --import-source on -k regex:k_tables_coz -s 1 -c 1 -o gpurun_out/prof_ml_tables_coz $CMDML > gpurun_out/ncu_ml.log 2>&1
CMDW8="python bench.py --custom 256,256,256,8 --steps 2 --warmup 1 --no-cpu-baseline --no-schoolbook --no-configs"
ncu --set full --clock-control none --import-source on -k regex:k_tables_gz -s 1 -c 1 -o gpurun_out/prof_w8_tables_gz $CMDW8 > gpurun_out/ncu_w8.log 2>&1
tail -3 gpurun_out/prof_round.log
