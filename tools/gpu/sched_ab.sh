# schedule variants of the pipelined batch (c2 bench line), alternated: default / all forward NTTs
# first / interleaved forward NTTs; with the timeline of one step each
for i in 1 2; do
  for cfg in "X=0" "HELINEAR_BATCH_FWD_FIRST=1" "HELINEAR_BATCH_INTERLEAVE=1"; do
    env $cfg timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 > /tmp/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$cfg', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
  done
done
for cfg in "HELINEAR_BATCH_FWD_FIRST=1" "HELINEAR_BATCH_INTERLEAVE=1"; do
  env $cfg HELINEAR_TIMELINE=1 python bench.py --no-cpu-baseline --no-attention --steps 1 --warmup 3 2>&1 >/dev/null | grep timeline | head -12 | sed "s/^/$cfg /"
done
