# full GPU test suite + sequential kernel times + the default bench line
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu/seq.sh
timeout 600 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], {k:d[k] for k in d if k in ('fc_local_share','client_gpu','rerandomized','attention_cross_terms')})"
