# GPU-box job: parity tests and timing of the whole-column row sort (default) against PCMM_ROWPERM_ALL=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or accumulator_exceptional or full_size_cussen or degenerate or signed_chain or general_fused or extreme or c64_config or tiny" > gpurun_out/t_rp.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/t_rp.log
CONFIGS="c256 c512 ml c64" STEPS=10 MODES="PCMM_ROWPERM_ALL=0" bash tools/gpu_iter.sh; cat gpurun_out/ab.log
