# split-mode batch: all 24 compute orders of the four c2 products, twice
python - <<'PY' > /tmp/orders.txt
import itertools
for p in itertools.permutations(range(4)): print(",".join(map(str,p)))
PY
for rep in $(seq 1 ${REPS:-2}); do
for o in $(cat /tmp/orders.txt); do
  HELINEAR_BATCH_SPLIT=1 HELINEAR_BATCH_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$o', d['value'])"
done
done
