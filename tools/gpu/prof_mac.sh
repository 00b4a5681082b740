timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mac_tc" -s 4 -c 4 -o gpurun_out/prof_mac python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_mac.log 2>&1; echo ncu=$?
