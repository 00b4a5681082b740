# new seeded e2e path: its GPU tests + one bench run (batch mode), printing the e2e block
timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -v -x -m gpu -k "seeded or linear_batch" > gpurun_out/e2e_pytest.log 2>&1; echo pytest rc=$?
grep -E "PASS|FAIL|ERROR|File" gpurun_out/e2e_pytest.log | head -30
timeout 400 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/e2e.json 2> gpurun_out/e2e.err; echo bench rc=$?
tail -3 gpurun_out/e2e.err
python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); print('value', d['value'], 'e2e', d['e2e'], d['clocks'])"
