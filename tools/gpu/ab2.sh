# A/B of two env settings (A="VAR=val ..." B="VAR=val ..."): GPU tests first, then the bench line
# sequential and pipelined, alternated twice
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
  for cfg in "$A" "$B"; do
    for mode in --sequential ""; do
      env $cfg timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 $mode > /tmp/ab.json 2>/dev/null
      python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$cfg', '$mode', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
    done
  done
done
