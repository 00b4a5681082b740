# pipelined c2 block under per-product tile sets (QKV; O; FF1; FF2), alternated
for rep in 1 2; do
for T in "16,8,32;8,8,64;16,8,32;4,32,32" "32,8,16;8,8,64;32,8,16;4,32,32" "32,8,16;8,8,64;32,8,16;8,16,32" "16,8,32;8,8,64;16,8,32;8,16,32" "32,4,32;8,8,64;32,4,32;8,16,32"; do
  timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 --tiles "$T" > /tmp/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$T', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
done
