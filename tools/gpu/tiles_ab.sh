# planned per-product tiles vs the single default tile: GPU tests, then bench sequential + pipelined
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
  for t in "" "--tile 16 8 32"; do
    for mode in --sequential ""; do
      timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 30 $t $mode > /tmp/ab.json 2>/tmp/ab.err || tail -5 /tmp/ab.err
      python -c "
import json; d=json.load(open('/tmp/ab.json')); print('tile=$t', '$mode', d['value'], d['roofline']['frac'], d['path_hbm_frac'], d['e2e']['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
    done
  done
done
