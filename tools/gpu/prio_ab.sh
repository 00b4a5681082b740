# forward-stream priority x submission order (pipelined bench line)
for i in 1 2; do
for p in 0 1 2; do for o in "" "0,1,2,3" "0,3,1,2"; do
  HELINEAR_FWD_PRIO=$p HELINEAR_BATCH_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('prio=$p order=$o', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done; done
