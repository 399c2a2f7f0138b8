#!/bin/bash
# A/B of prebuilt libpcmm variants in ${VARDIR:-variants}/: GPU field/point tests, bench configs, NEXT-2 tool
cp paper_2504_14497_b200/libpcmm.so /tmp/lib_orig.so
for v in ${VARDIR:-variants}/*.so; do
  cp $v paper_2504_14497_b200/libpcmm.so
  touch paper_2504_14497_b200/libpcmm.so
  r=$(python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -W ignore -k "field or point or c64 or tiny or bsgs or comb or decrypt" 2>&1 | tail -1)
  echo "== $v : $r"
  CONFIGS="${CONFIGS:-c256}" bash tools/bench_all.sh
  python tools/next2_bench.py 2>/dev/null | grep -i "encrypt\|BSGS, s = 2^22"
done
cp /tmp/lib_orig.so paper_2504_14497_b200/libpcmm.so
