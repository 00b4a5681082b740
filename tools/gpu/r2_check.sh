# round-2 check: GPU tests, smoke, default bench line
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print({k: d.get(k) for k in ('value','ms_per_step','e2e','roofline')})" 2>&1 | head -5
