# quick: GPU tests (-x) + bench line sequential and pipelined (30 steps)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for mode in --sequential "" --sequential ""; do
  timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 $mode > /tmp/ab.json 2>/tmp/ab.err || tail -5 /tmp/ab.err
  python -c "
import json; d=json.load(open('/tmp/ab.json')); print('$mode', d['value'], round(d['roofline']['frac'],3), round(d['path_hbm_frac'],3), d['e2e']['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
