timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu/seq.sh
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo bench batch rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_b.json')); print(d['value'], d['roofline']['frac'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
