#!/bin/bash
# schoolbook step time per config (GPU box): python bench.py --path schoolbook (no CPU leg)
for c in ${CONFIGS:-c256}; do
  python bench.py --config $c --path schoolbook --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-schoolbook 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c schoolbook', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d.get('kernels',{}).items()})"
done
