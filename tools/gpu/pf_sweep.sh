for i in 1 2; do for pf in 0 2 4 8; do for mode in --sequential ""; do
  HELINEAR_MAC_PF=$pf timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 $mode > /tmp/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/sw.json')); print('pf=$pf $mode', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done; done
