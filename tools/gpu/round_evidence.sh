# Full evidence pass (round 2): smoke, GPU tests, bench lines (c2 default + shard path + reference arm,
# c3 and c4 stacks), ncu launch list + full captures, compute-sanitizer.  Outputs in gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err; echo bench=$?
timeout 300 python bench.py --mode shard --no-cpu-baseline --no-attention > gpurun_out/ev/bench_c2_shard.json 2> gpurun_out/ev/bench_c2_shard.err; echo shard=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_c2_reference.json 2> gpurun_out/ev/bench_c2_reference.err; echo ref=$?
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err; echo c3=$?
timeout 1800 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err; echo c4=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/ev/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mac_tc|k_ntt_fwd|k_c1_|k_ntt_inv_mask|k_intt_c0" -s 36 -c 24 --csv --log-file gpurun_out/ev/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/ev/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mac_tc" -s 12 -c 4 -o gpurun_out/ev/prof_mac_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/ev/ncu2.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ntt_fwd_c0x2|k_intt_c0_pruned" -s 8 -c 4 -o gpurun_out/ev/prof_ntt_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/ev/ncu3.log 2>&1; echo ncu3=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mac_tc" -s 8 -c 2 -o gpurun_out/ev/prof_mac_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ev/ncu4.log 2>&1; echo ncu4=$?
bash tools/gpu/sanitize.sh > gpurun_out/ev/sanitize_summary.txt 2>&1; echo sanitize=$?
mv gpurun_out/sanitize_*.log gpurun_out/ev/ 2>/dev/null
