# A/B of prebuilt libraries build/libs/{base,$VARIANTS}.so on c2 (pipelined) and the c3/c4 stacks
L=paper_2305_18396_b200/lib/libhelinear.so
for v in base ${VARIANTS}; do
  cp build/libs/$v.so $L
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-attention > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v c2', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
  for c in ${CFGS:-c3 c4}; do
    timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v $c', d['value'], d['ms_per_block'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
  done
done
cp build/libs/base.so $L
