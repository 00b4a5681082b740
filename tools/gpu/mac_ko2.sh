for ko in 0 1 8; do
HELINEAR_MAC_KO=$ko timeout 300 python bench.py --no-cpu-baseline --sequential --steps 20 > gpurun_out/ko.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ko.json')); print('ko=$ko', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
