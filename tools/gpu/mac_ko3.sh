for ko in 0 1 4 7; do
HELINEAR_MAC_KO=$ko timeout 300 python bench.py --no-cpu-baseline --no-attention --sequential --steps 20 > gpurun_out/ko.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ko.json')); print('ko=$ko', d['value'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
HELINEAR_MAC_PROF=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-attention --sequential 2>&1 | grep mac_tc | tail -4
