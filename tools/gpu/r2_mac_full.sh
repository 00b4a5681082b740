# ncu --set full with source of one tensor-core MAC launch on c4 (and c3)
for c in ${CFGS:-c4 c3}; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_mac_tc' -c 1 -o gpurun_out/mac_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2> gpurun_out/mac_$c.err
done
