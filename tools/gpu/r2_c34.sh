timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or serial or engine or full_size or fused or shard" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel.log
for c in c3 c4; do
timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$c', d['value'], d['ms_per_block'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['config']['tile'])" || tail -3 /tmp/c.err
done
HELINEAR_MAC_PROF=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/prof_c3.err > /dev/null; grep mac_tc gpurun_out/prof_c3.err | sort | uniq | awk 'NR%12==1' | head -8
