for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log; done
CFGS="c3" bash tools/gpu/r2_quick.sh 2>&1 | grep -v pytest
