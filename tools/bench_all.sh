#!/bin/bash
# quick per-config bench summary (GPU box)
for c in ${CONFIGS:-c256 c512 ml c64}; do
  python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-schoolbook | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$c', round(d['ms_per_step'],3), 'roof(accum)', round(d['roofline']['frac'],3), 'roof(step)', round(d['roofline_whole_step']['frac'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
