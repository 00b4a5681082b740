# MAC ring budget in the pipelined batch (HELINEAR_BATCH_MAC_SMEM_KB), alternated twice
for rep in 1 2; do
for kb in ${KBS:-140 155 170 185 200}; do
  HELINEAR_BATCH_MAC_SMEM_KB=$kb timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 > /tmp/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$kb', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
done
