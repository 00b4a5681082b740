timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or serial or engine or full_size" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel.log
timeout 600 python bench.py --config c3 --steps 2 --warmup 2 --no-cpu-baseline > /tmp/c.json 2>/tmp/c.err; python -c "
import json; d=json.load(open('/tmp/c.json')); print('c3', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/c.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-attention --sequential > /dev/null 2>&1; echo seq=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ntt_fwd_c0x2|k_intt_c0_pruned" -s 8 -c 4 -o gpurun_out/prof_ntt_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/ncu_ntt.log 2>&1; echo ncu=$?
