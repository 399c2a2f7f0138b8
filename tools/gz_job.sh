# GPU-box job: forced-mode parity tests of k_tables_gz (PCMM_TABLES_GZ=2) and its timing against
# k_tables / k_tables_x + k_affine (PCMM_TABLES_GZ=0/1/2) on 64^3, tiny, ML and the w = 8 / w = 6 custom shapes
mkdir -p gpurun_out
PCMM_TABLES_GZ=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or tiny or c64_config or degenerate or consecutive_column or signed_chain or xyzz_level1 or all_identity or extreme or plan_matches or vector_times" > gpurun_out/t_gz.log 2>&1
echo "rc=$?" >> gpurun_out/t_gz.log
tail -12 gpurun_out/t_gz.log
for mode in 0 1 2; do
  echo "== GZ=$mode"
  PCMM_TABLES_GZ=$mode CONFIGS="c64 tiny ml" STEPS=10 bash tools/bench_all.sh
  for c in "64,64,64,8" "256,256,256,8" "128,128,128,6"; do
    PCMM_TABLES_GZ=$mode python bench.py --custom $c --steps 5 --warmup 3 --no-cpu-baseline --no-schoolbook --no-configs | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
done
