# ncu launch list (durations, DRAM bytes) of the first block items of the c3 and c4 stacks
for c in ${CFGS:-c3 c4}; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_ntt_fwd_c0x2|k_c1_tx16|k_mac_tc|k_intt_c0" -c ${NK:-30} --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_$c.err
python tools/ncu_summary.py launches gpurun_out/launches_$c.csv > gpurun_out/launches_${c}_summary.txt
done
