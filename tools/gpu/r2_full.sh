# full GPU suite + c2/c3/c4 bench summaries (round 2 iteration loop)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_full.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-attention > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('c2', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
for c in ${CFGS:-c3 c4}; do
timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$c', d['value'], d['ms_per_block'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
done
