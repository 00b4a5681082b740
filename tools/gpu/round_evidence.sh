# full evidence pass: GPU tests, smoke, bench line (+cpu baseline), shard mode, ncu launch list, ncu full capture
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python bench.py --mode shard --no-cpu-baseline > gpurun_out/bench_shard.json 2> gpurun_out/bench_shard.err; echo shard=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
# the larger BASELINE configs (parity-test cases, measured for context): one block each at the planner's tiles
for c in c3 c4; do timeout 600 python bench.py --config $c --plan --sequential --no-cpu-baseline --no-attention --steps 5 > gpurun_out/bench_${c}_plan_seq.json 2> gpurun_out/bench_${c}.err; echo $c=$?; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mac_tc|k_ntt_fwd_c0|k_c1_out|k_ntt_inv_mask|k_intt_c0" -s 36 -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"k_mac_tc|k_ntt_fwd_c0|k_c1_out|k_ntt_inv_mask|k_intt_c0" -s 12 -c 12 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
