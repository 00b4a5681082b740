timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-attention > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('c2', d['value'], {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()})"
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo c3plain=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_mac_tc -s 8 -c 4 -o gpurun_out/prof_mac_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_c3.log
