# c2 A/B of prebuilt variants (VARIANTS), REPS rounds alternating
L=paper_2305_18396_b200/lib/libhelinear.so
cp $L /tmp/orig.so
for rep in $(seq ${REPS:-3}); do
for v in ${VARIANTS:-cur}; do
  cp build/libs/$v.so $L
  timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 ${ARGS} > /tmp/c.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
done
cp /tmp/orig.so $L
