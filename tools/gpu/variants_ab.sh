# A/B of prebuilt library variants build/libs/<v>.so (VARIANTS="base wnorm ..."): c3 stack (+ c2 if C2=1)
L=paper_2305_18396_b200/lib/libhelinear.so
cp $L /tmp/orig.so
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  cp build/libs/$v.so $L
  timeout 600 python bench.py --config ${CFG:-c3} --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v ${CFG:-c3}', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -2 /tmp/c.err
  if [ "$C2" = 1 ]; then timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/c.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v c2', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; fi
done
done
cp /tmp/orig.so $L
