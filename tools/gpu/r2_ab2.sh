timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or serial or engine or full_size or fused or shard" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel.log
VARIANTS="zmma nozmma" bash tools/gpu/variants_ab.sh
VARIANTS="zmma nozmma" CFG=c4 bash tools/gpu/variants_ab.sh 2>&1 | head -2
