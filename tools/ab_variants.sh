#!/bin/bash
# A/B: run quick parity + c256 bench for each prebuilt libpcmm variant in variants/
cp paper_2504_14497_b200/libpcmm.so /tmp/lib_orig.so
for v in ${VARDIR:-variants}/*.so; do
  cp $v paper_2504_14497_b200/libpcmm.so
  touch paper_2504_14497_b200/libpcmm.so
  r=$(python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -W ignore -k "c64 or field or ragged" 2>&1 | tail -1)
  echo "== $v : $r"
  CONFIGS="${CONFIGS:-c256}" bash tools/bench_all.sh
done
cp /tmp/lib_orig.so paper_2504_14497_b200/libpcmm.so
