timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/plain.log 2>&1; echo plain=$?
grep "ncu --metrics" tools/gpu/round_evidence.sh | bash
