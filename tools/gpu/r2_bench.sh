# bench lines: c2 default, c2 shard mode at N=1, c3 stack, c4 stack (one GPU)
timeout 600 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python bench.py --mode shard --steps 10 --no-cpu-baseline --no-attention > gpurun_out/bench_shard.json 2> gpurun_out/bench_shard.err; echo shard=$?
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
for f in bench bench_shard bench_c3 bench_c4; do python -c "
import json,sys; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('ms_per_block'), d['e2e']['value'], d.get('path_roofline'), {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()}, d.get('cpu_baseline',{}).get('value'))" 2>&1 | tail -1; tail -2 gpurun_out/$f.err; done
