# A/B: the batch bench line of wt_old (an older build) vs the current tree, alternated
for i in 1 2; do
  for d in wt_old .; do
    (cd $d && timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$d', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})")
  done
done
