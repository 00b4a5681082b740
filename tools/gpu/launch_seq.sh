# ncu launch list (durations, DRAM bytes) of one sequential block step, after the plain run exits 0
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" -s 60 -c 22 --csv --log-file gpurun_out/launches_seq.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/ncu1.log 2>&1; echo ncu=$?
