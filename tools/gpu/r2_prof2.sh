# role profiling of the tensor-core MAC on c3 and c4 (needs the -DHL_MAC_PROF build in build/libs/prof.so)
L=paper_2305_18396_b200/lib/libhelinear.so; cp $L /tmp/orig.so; cp build/libs/prof.so $L
for c in ${CFGS:-c3 c4}; do
HELINEAR_MAC_PROF=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/prof_$c.err > /dev/null; grep mac_tc gpurun_out/prof_$c.err | awk -F']' '!seen[$1]++' | head -8
done
cp /tmp/orig.so $L
