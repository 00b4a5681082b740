for i in 1 2; do for kb in 155 175 190; do
  HELINEAR_BATCH_MAC_SMEM_KB=$kb timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/sw.json')); print('kb=$kb', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done
