#!/bin/bash
# perm_search.sh LISTFILE: each line "name flags..." -> abv/name.so (hot.cu recompiled with the flags,
# linked with the default build's other objects); up to 8 compilations at a time.  The k_accum loop's
# schedule (and time) changes with the source order of its ten products although the arithmetic does
# not; this builds the candidates that tools/gpu_iter.sh then times on the GPU box.
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2504_14497_b200 import build as b; b.build()"
mkdir -p abv /tmp/perm
B=paper_2504_14497_b200/_build
C=paper_2504_14497_b200/csrc
build_one() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -I include "$@" -c $C/hot.cu -o /tmp/perm/$name.o && \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o abv/$name.so /tmp/perm/$name.o $B/kernels.o $B/affine.o $B/taff.o $B/tgz.o $B/school.o $B/strassen.o $B/wide.o $B/next2.o $B/paillier.o $B/api.o
}
n=0
while read -r name flags; do
  [ -z "$name" ] && continue
  build_one $name $flags &
  n=$((n+1))
  if [ $((n % 8)) -eq 0 ]; then wait; fi
done < "$1"
wait
ls -la abv
