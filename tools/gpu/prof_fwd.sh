# ncu full capture of the forward-side kernels of one QKV product (sequential bench)
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:"k_ntt_fwd_c0|k_c1_to_x|k_ntt_inv_mask|k_intt_c0" -s 8 -c 8 -o gpurun_out/prof_fwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-attention --sequential > gpurun_out/ncu_fwd.log 2>&1; echo ncu=$?
