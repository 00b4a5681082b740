timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or serial or engine or full_size or fused or shard or general" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-attention > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('c2', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
for c in ${CFGS:-c3 c4}; do
timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('$c', d['value'], d['ms_per_block'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
done
[ "$PROF" = 1 ] && bash tools/gpu/r2_prof.sh | head -3
