# batch pipeline variants (pipelined bench line only), alternated twice
for i in 1 2; do
  for cfg in "HELINEAR_BATCH_KEEP_ORDER=1" "X=1" "HELINEAR_BATCH_SPLIT=1" "HELINEAR_BATCH_SPLIT=1 HELINEAR_BATCH_KEEP_ORDER=1"; do
    env $cfg timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$cfg', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
  done
done
