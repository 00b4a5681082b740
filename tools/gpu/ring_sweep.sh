# batch pipeline: MAC ring budget sweep (pipelined bench line)
for kb in 120 150 157 165 190 227; do
  HELINEAR_BATCH_MAC_SMEM_KB=$kb timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/sw.json')); print('kb=$kb', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
