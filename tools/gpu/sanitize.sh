# compute-sanitizer passes over c0 / c1 / a fat CW=16 product through he_matmul_share, he_linear_batch
# and he_linear_batch_host (tools/gpu/sanitize_run.py checks every result against the oracle)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for w in c0 c1 fat; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/gpu/sanitize_run.py $w > gpurun_out/sanitize_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok|MISMATCH' gpurun_out/sanitize_${tool}_${w}.log | tr '\n' ' ' | cut -c1-300)"
  done
done
