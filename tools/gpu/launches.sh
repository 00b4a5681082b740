timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sequential > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_seq.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sequential > gpurun_out/ncu1.log 2>&1; echo ncu=$?
