# batch pipeline: MAC grid x MAC ring smem sweep (SM partition between the MAC and the NTT kernels)
for kb in 150 227; do for g in 148 132 116 100 84; do
HELINEAR_BATCH_MAC_GRID=$g HELINEAR_BATCH_MAC_SMEM_KB=$kb timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/sw.json 2>/dev/null
python -c "
import json; d=json.load(open('/tmp/sw.json')); print('kb=$kb grid=$g', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done
