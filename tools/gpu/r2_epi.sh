timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-attention > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('c2', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
for c in c3 c4; do
timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$c', d['value'], d['ms_per_block'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
done
HELINEAR_MAC_PROF=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/prof_c3.err > /dev/null; grep mac_tc gpurun_out/prof_c3.err | sort | uniq | awk 'NR%12==1' | head -8
