# converter rewrite: parity + c2 + c3/c4 stacks
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-attention > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
HELINEAR_MAC_PROF=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/prof_c3.err > /dev/null; grep mac_tc gpurun_out/prof_c3.err | sort | uniq -c | sort -rn | head -8
for f in bench bench_c3 bench_c4; do python -c "
import json,sys; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('ms_per_block'), d['e2e']['value'], d.get('path_roofline',{}).get('frac'), d.get('roofline',{}).get('frac'), {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()})" 2>&1 | tail -1; tail -2 gpurun_out/$f.err; done
