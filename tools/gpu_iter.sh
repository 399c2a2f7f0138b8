#!/bin/bash
# One GPU iteration (run under gpurun): a pytest subset (TESTK, a -k expression; empty = skip), then
# per-config kernel times (tools/bench_all.sh) for the default library, each abv/*.so variant and each
# MODES entry ("ENV=VALUE" strings, run on the default library).  Output under gpurun_out/.
mkdir -p gpurun_out
if [ -n "$TESTK" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -W ignore -k "$TESTK" > gpurun_out/tests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/tests.log
fi
CONFIGS="${CONFIGS:-c256}" STEPS=${STEPS:-10} bash tools/bench_all.sh > gpurun_out/ab.log 2>&1
echo "== default" >> gpurun_out/ab.log
for m in $MODES; do
  env $m CONFIGS="${CONFIGS:-c256}" STEPS=${STEPS:-10} bash tools/bench_all.sh >> gpurun_out/ab.log 2>&1
  echo "== $m" >> gpurun_out/ab.log
done
if ls abv/*.so > /dev/null 2>&1; then
  cp paper_2504_14497_b200/libpcmm.so /tmp/lib_orig.so
  for v in abv/*.so; do
    cp $v paper_2504_14497_b200/libpcmm.so; touch paper_2504_14497_b200/libpcmm.so
    CONFIGS="${CONFIGS:-c256}" STEPS=${STEPS:-10} bash tools/bench_all.sh >> gpurun_out/ab.log 2>&1
    echo "== $v" >> gpurun_out/ab.log
  done
  cp /tmp/lib_orig.so paper_2504_14497_b200/libpcmm.so; touch paper_2504_14497_b200/libpcmm.so
fi
