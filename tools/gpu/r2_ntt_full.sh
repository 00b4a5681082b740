# ncu --set full with source of the forward NTT and pruned inverse on c3 (N=4096) and c4 (N=8192)
for c in c3 c4; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_ntt_fwd_c0x2|k_intt_c0_pruned' -c 2 -o gpurun_out/ntt_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2> gpurun_out/ntt_$c.err
done
