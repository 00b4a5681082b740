for kb in 100 125 150 175 227; do for G in 1 2; do
HELINEAR_NTT_G=$G HELINEAR_BATCH_MAC_SMEM_KB=$kb timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/sw.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('kb=$kb G=$G', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done
