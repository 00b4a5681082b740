# Full evidence pass (round 2), part B: ncu launch list (c2 step) + full captures of the MAC (c2, c3)
# and of the NTT kernels (c2); the reports are summarised to CSV on the box (the .ncu-rep of the c2
# MAC is kept: profiles/traffic.json is derived from it)
set -x
mkdir -p gpurun_out/evn
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/evn/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mac_tc|k_ntt_fwd|k_c1_|k_ntt_inv_mask|k_intt_c0" -s 36 -c 24 --csv --log-file gpurun_out/evn/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/evn/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_mac_tc" -s 12 -c 4 -o gpurun_out/evn/prof_mac_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention > gpurun_out/evn/ncu2.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_ntt_fwd_c0x2|k_intt_c0_pruned" -s 8 -c 4 -o /tmp/prof_ntt_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/evn/ncu3.log 2>&1; echo ncu3=$?
ncu -i /tmp/prof_ntt_c2.ncu-rep --page raw --csv > gpurun_out/evn/prof_ntt_c2_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:"k_mac_tc" -s 8 -c 2 -o /tmp/prof_mac_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/evn/ncu4.log 2>&1; echo ncu4=$?
ncu -i /tmp/prof_mac_c3.ncu-rep --page raw --csv > gpurun_out/evn/prof_mac_c3_raw.csv 2>/dev/null
ncu -i gpurun_out/evn/prof_mac_c2.ncu-rep --page raw --csv > gpurun_out/evn/prof_mac_c2_raw.csv 2>/dev/null
du -sh gpurun_out; ls -la gpurun_out/evn
