# A/B of the default library and each abv/*.so on the w = 8 / w = 6 custom shapes (k_tables_gz)
run() {
  for c in "256,256,256,8" "128,128,128,6"; do
    python bench.py --custom $c --steps 5 --warmup 3 --no-cpu-baseline --no-schoolbook --no-configs | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
}
echo "== default"; run
if ls abv/*.so > /dev/null 2>&1; then
  cp paper_2504_14497_b200/libpcmm.so /tmp/lib_orig.so
  for v in abv/*.so; do
    cp $v paper_2504_14497_b200/libpcmm.so; touch paper_2504_14497_b200/libpcmm.so
    echo "== $v"; run
  done
  cp /tmp/lib_orig.so paper_2504_14497_b200/libpcmm.so
fi
