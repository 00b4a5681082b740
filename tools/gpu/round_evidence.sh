# Full evidence pass (round 2), part A: smoke, GPU tests, bench lines (c2 default + shard path +
# reference arm, c3 and c4 stacks), compute-sanitizer.  Outputs in gpurun_out/ev/ (text only).
set -x
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err; echo bench=$?
timeout 300 python bench.py --mode shard --no-cpu-baseline --no-attention > gpurun_out/ev/bench_c2_shard.json 2> gpurun_out/ev/bench_c2_shard.err; echo shard=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_c2_reference.json 2> gpurun_out/ev/bench_c2_reference.err; echo ref=$?
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err; echo c3=$?
timeout 1800 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err; echo c4=$?
bash tools/gpu/sanitize.sh > gpurun_out/ev/sanitize_summary.txt 2>&1; echo sanitize=$?
mv gpurun_out/sanitize_*.log gpurun_out/ev/ 2>/dev/null
du -sh gpurun_out
