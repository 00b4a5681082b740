timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for G in 2 4 1; do
HELINEAR_NTT_G=$G timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$G.json 2> gpurun_out/bench_g$G.err; echo bench G=$G rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_g$G.json')); print(d['value'], d['roofline']['frac'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
