# GPU-box job: split-k sweep (PCMM_KSPLIT) of the accumulate kernel on 256^3, 512^3 and ML
for ks in 1 2; do echo "== c256 ks=$ks"; PCMM_KSPLIT=$ks CONFIGS="c256" STEPS=10 bash tools/bench_all.sh; done
for ks in 1 2 3; do echo "== c512 ks=$ks"; PCMM_KSPLIT=$ks CONFIGS="c512" STEPS=6 bash tools/bench_all.sh; done
for ks in 4 5 6 8; do echo "== ml ks=$ks"; PCMM_KSPLIT=$ks CONFIGS="ml" STEPS=10 bash tools/bench_all.sh; done
