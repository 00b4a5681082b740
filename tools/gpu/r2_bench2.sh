timeout 600 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
for f in bench bench_c4; do python -c "
import json,sys; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('ms_per_block'), d['e2e'], d.get('path_roofline'), d.get('roofline'), {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()}, d.get('cpu_baseline',{}).get('value'), d['config'].get('tile_choice'))" 2>&1 | tail -1; tail -2 gpurun_out/$f.err; done
