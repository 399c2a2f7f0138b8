timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or accumulator_exceptional or full_size_cussen or degenerate or signed_chain or general_fused or extreme or c64_config or tiny or wide_every or accumulate_modes_forced" 2>&1 | tail -2
CONFIGS="c256 c512 ml c64 tiny" STEPS=10 bash tools/bench_all.sh
for c in 256,256,256,8 256,256,256,12; do python bench.py --custom $c --steps 5 --warmup 3 --no-cpu-baseline --no-schoolbook --no-configs | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
