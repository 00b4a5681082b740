set -x
timeout 120 python -m pytest tests -m gpu -x -q -k "engines_bit_exact and 2" > gpurun_out/pt_tc1.log 2>&1; echo first=$?
tail -5 gpurun_out/pt_tc1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo bench=$?
cat gpurun_out/bench_tc.json
