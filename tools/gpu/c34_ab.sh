# A/B of an env setting on the larger configs (planner tiles, sequential, one block)
for cfg in "$A" "$B"; do
  for c in c3 c4; do
    env $cfg timeout 600 python bench.py --config $c --plan --sequential --no-cpu-baseline --no-attention --steps 3 --warmup 3 > /tmp/c.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/c.json')); print('$cfg', '$c', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
done
