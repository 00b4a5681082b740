for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --sequential --steps 30 > gpurun_out/seq.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/seq.json')); print('seq', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
