for rep in 1 2 3; do
for o in ${ORDERS:-0,1,2,3 1,2,0,3 1,0,2,3}; do
  HELINEAR_BATCH_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 > /tmp/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$o', d['value'])"
done
done
