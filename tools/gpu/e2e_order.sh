for o in ${ORDERS:-2,0,3,1 1,2,3,0 1,0,2,3 1,3,2,0 1,2,0,3 1,0,3,2 1,2,0,3}; do
  BENCH_E2E_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 20 > /tmp/e.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/e.json')); print('$o', d['value'], d['e2e']['value'])"
done
