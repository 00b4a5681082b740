# converter change A/B: c3 MAC role profile + c3/c2 sequential lines
HELINEAR_MAC_PROF=1 python bench.py --config c3 --plan --sequential --no-cpu-baseline --no-attention --steps 1 --warmup 0 2>&1 >/dev/null | grep mac_tc | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in c3 c2; do
  timeout 600 python bench.py --config $c --plan --sequential --no-cpu-baseline --no-attention --steps 5 > /tmp/c.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('$c seq', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 > /tmp/c.json 2>/dev/null
python -c "
import json; d=json.load(open('/tmp/c.json')); print('c2 pipelined', d['value'])"
