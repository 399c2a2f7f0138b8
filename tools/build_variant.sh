#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS": build libpcmm.so with extra nvcc flags into abv/NAME.so,
# then rebuild the default library (measurement-only builds for A/B runs on the GPU box)
set -e
cd "$(dirname "$0")/.."
mkdir -p abv
PCMM_EXTRA_NVCC_FLAGS="$2" python -c "from paper_2504_14497_b200 import build as b; b.build(force=True)"
cp paper_2504_14497_b200/libpcmm.so "abv/$1.so"
python -c "from paper_2504_14497_b200 import build as b; b.build(force=True)"
