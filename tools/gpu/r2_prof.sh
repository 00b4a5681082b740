# role profiling of the tensor-core MAC: needs the -DHL_MAC_PROF build in build/libs/prof.so
L=paper_2305_18396_b200/lib/libhelinear.so; cp $L /tmp/orig.so; cp build/libs/prof.so $L
HELINEAR_MAC_PROF=1 timeout 600 python bench.py --config ${CFG:-c3} --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/prof_${CFG:-c3}.err > /dev/null; grep mac_tc gpurun_out/prof_${CFG:-c3}.err | sort | uniq | awk 'NR%12==1' | head -8
cp /tmp/orig.so $L
