timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); print(d['value'], d['roofline']['frac'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
HELINEAR_MAC_PROF=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep mac_tc | tail -4
