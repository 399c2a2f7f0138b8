# GPU-box job: parity tests under PCMM_ACC_MODE=2, 3 and the accumulate modes' timing (DESIGN.md section 6 table)
mkdir -p gpurun_out
for mode in 2 3; do
PCMM_ACC_MODE=$mode timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or accumulator_exceptional or full_size_cussen or degenerate or signed_chain or general_fused or extreme" > gpurun_out/t_acc$mode.log 2>&1
echo "mode $mode rc=$?"; tail -2 gpurun_out/t_acc$mode.log
done
CONFIGS="c256 c512 ml" STEPS=10 MODES="PCMM_ACC_MODE=1 PCMM_ACC_MODE=2 PCMM_ACC_MODE=3" bash tools/gpu_iter.sh; cat gpurun_out/ab.log
for mode in 0 2 3; do
  PCMM_ACC_MODE=$mode python bench.py --custom 256,256,256,8 --steps 5 --warmup 3 --no-cpu-baseline --no-schoolbook --no-configs | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('w8 mode $mode', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
