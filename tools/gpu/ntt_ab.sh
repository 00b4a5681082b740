# A/B of an env-selected kernel variant: GPU tests with the new default, then the bench line
# sequential and pipelined with VAR=0 / VAR=1 (VAR defaults to HELINEAR_NTT_P)
VAR=${VAR:-HELINEAR_NTT_P}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
  for v in 0 1; do
    for mode in --sequential ""; do
      env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 $mode > /tmp/ab.json 2>/dev/null
      python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$VAR=$v', '$mode', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
    done
  done
done
